// Internal helpers shared by the translation units of libsfft (not exported).
#pragma once

#include <string>

// Record `msg` as this thread's sfft_last_error() and return `code`.
int sfft_internal_fail(int code, const std::string& msg);
