/*
 * sfft.h -- C ABI of the B200-native batched C2C FFT (sm_100a).
 *
 * This is the drop-in boundary for the reference's plan/execute hot path
 * (/root/reference/pkg/src/stagefft).  The reference has no native code and
 * no FFI; every entry point below names the Python interface it replaces, so
 * a maintainer can bind it with ctypes:
 *
 *   sfft_plan_create    <- make_plan            planner.py:139-188
 *                          (+ factorize_stages  planner.py:38-59,
 *                             build_twiddle_table numerics.py:55-71)
 *   sfft_execute        <- execute / execute_timed  executor.py:50-96, batched
 *                          like FourierTransformer._apply estimator.py:61-68
 *   sfft_execute_host   <- the same call on host buffers (numpy in, numpy out)
 *   sfft_plan_destroy   <- FftPlan lifetime     planner.py:92-136
 *   sfft_plan_info      <- FftPlan fields (stages, chunk) planner.py:107-114
 *   sfft_plan_twiddles  <- FftPlan.twiddles.factors numerics.py:41-52
 *   status codes        <- errors.py:9-34 exception tree
 *
 * Conventions: plain pointers and sizes only; interleaved complex
 * (float2 / double2), rows of n contiguous elements, row-major batch.  No C++
 * exception crosses this boundary; every function returns an SFFT_* status
 * and sfft_last_error() returns a thread-local message for the last failure.
 */
#ifndef SFFT_H_
#define SFFT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes -- one per reference exception class (errors.py:9-34) */
#define SFFT_OK 0
#define SFFT_ERR_INVALID_LENGTH 1     /* InvalidLengthError   errors.py:13-14 */
#define SFFT_ERR_UNSUPPORTED_LENGTH 2 /* UnsupportedLengthError errors.py:17-18 */
#define SFFT_ERR_PLAN 3               /* PlanError            errors.py:21-22 */
#define SFFT_ERR_SHAPE 4              /* ShapeError           errors.py:25-26 */
#define SFFT_ERR_DOMAIN 5             /* DomainError (NaN/Inf input) errors.py:29-30 */
#define SFFT_ERR_CUDA 6               /* device/runtime failure (no reference analogue) */
#define SFFT_ERR_ARGUMENT 7           /* null/misaligned pointer, bad enum (FftError) */

#define SFFT_SINGLE 0 /* complex64  (float2)  -- the reference engine dtype */
#define SFFT_DOUBLE 1 /* complex128 (double2) -- new precision axis          */

#define SFFT_FORWARD 0 /* Direction.FORWARD planner.py:29 */
#define SFFT_INVERSE 1 /* Direction.INVERSE planner.py:30, scaled by 1/n */

#define SFFT_MIN_LENGTH 2
#define SFFT_MAX_LENGTH 2048

#define SFFT_KERNEL_STOCKHAM 0 /* G=n/R threads per sequence, smem exchange */
#define SFFT_KERNEL_TILE 1     /* thread per sequence, warp-staged tile     */
#define SFFT_KERNEL_SPLIT2 2   /* two one-warp half transforms + radix-2    */
#define SFFT_KERNEL_FOURSTEP 3 /* 32 x 64 four-step, shuffle radix-2, fp64 N=2048 */

typedef struct sfft_plan* sfft_plan_t;

typedef struct sfft_plan_info {
  int32_t n;
  int32_t precision;
  int32_t direction;
  int32_t device;
  int64_t batch;               /* batch the plan was created for (0 = any) */
  int32_t kernel;              /* SFFT_KERNEL_* */
  int32_t elems_per_thread;    /* R (stockham) or n (tile) */
  int32_t seqs_per_cta;        /* sequences one CTA owns */
  int32_t threads_per_cta;
  int32_t smem_bytes;          /* dynamic shared memory per CTA */
  int32_t num_passes;          /* radix passes of the GPU schedule */
  int32_t radices[8];          /* GPU pass radices, first to last */
  int64_t twiddle_elems;       /* per-pass twiddle table length (elements) */
  int32_t variant;             /* index into the kernel variant table */
  int32_t layout;              /* stockham smem layout: 1 padded, 2 row swizzle, 3 split re/im exchange (fp64) */
  int32_t twiddle_policy;      /* 0: every twiddle loaded; 1: powers of two + products */
  int32_t loader;              /* 0: per-thread global loads; 1: one bulk TMA copy per CTA;
                                  2: persistent CTAs, pipelined bulk TMA copies;
                                  3: one bulk TMA copy + gathers through tensor memory;
                                  4: as 3, the staging gather only */
  int32_t smem_carveout;       /* preferred shared-memory carveout, % of max (-1: driver default) */
  int32_t pipeline_stages;     /* loader 2: shared-memory stage buffers per CTA (else 0) */
  int32_t real_input;          /* 1: SFFT_INPUT_REAL is supported (sfft_execute_ex) */
  int32_t real_loader;         /* loader of the real-input kernel (same passes, so the same
                                  results as widening; the loader may differ) */
} sfft_plan_info_t;

/* Library version (major*10000 + minor*100 + patch). */
int sfft_version(void);

/* Number of kernel variants compiled for (n, precision); variant 0 is the
 * default the planner picks.  Returns 0 for an unsupported pair. */
int sfft_num_variants(int32_t n, int32_t precision);

/* build_twiddle_table (numerics.py:55-71) on the host, no device needed:
 * n complex values of `precision`, angle (-2*pi/n)*k in double, rounded once
 * for single, factors[0] = 1 exactly.  n power of two in [1, 4096]. */
int sfft_build_twiddle_table(int32_t n, int32_t precision, void* host_out,
                             int64_t capacity_bytes);

/* Geometry of kernel variant `variant` for (n, precision) without creating a
 * plan or touching a device (direction/device/batch fields are zero). */
int sfft_variant_info(int32_t n, int32_t precision, int32_t variant, sfft_plan_info_t* info);

/* make_plan: validate (n power of two in [2, 2048]), choose the kernel,
 * build the twiddle table in double (rounded once for single), upload the
 * per-pass table to `device`.  batch >= 0 (0 = unspecified). */
int sfft_plan_create(sfft_plan_t* plan, int32_t n, int32_t precision, int32_t direction,
                     int64_t batch, int32_t device);

/* Same, forcing a kernel variant (0 .. sfft_num_variants-1); for tuning. */
int sfft_plan_create_variant(sfft_plan_t* plan, int32_t n, int32_t precision,
                             int32_t direction, int64_t batch, int32_t device,
                             int32_t variant);

int sfft_plan_destroy(sfft_plan_t plan);

int sfft_plan_info(sfft_plan_t plan, sfft_plan_info_t* info);

/* Copy the plan's base twiddle table (n complex values of the plan precision,
 * factors[k] = exp(-2*pi*i*k/n), factors[0] = 1) to host memory. */
int sfft_plan_twiddles(sfft_plan_t plan, void* host_out, int64_t capacity_bytes);

/* Asynchronous batched execute on device memory, out-of-place or in-place
 * (d_in == d_out).  `batch` rows of n elements; batch == 0 is a no-op.
 * `stream` is a cudaStream_t (NULL = legacy default stream).  If
 * `d_nonfinite` is non-NULL the kernel ORs 1 into it when any input value is
 * NaN/Inf (the caller zeroes it and reads it after the stream completes).
 * Alignment: 16 bytes for both pointers.  Buffers are either disjoint or
 * identical (complex input in place); any other overlap -- a shifted view,
 * or real input (_ex) sharing memory with its complex output -- returns
 * SFFT_ERR_ARGUMENT (the same rule holds for every execute entry point). */
int sfft_execute(sfft_plan_t plan, const void* d_in, void* d_out, int64_t batch, void* stream,
                 int32_t* d_nonfinite);

/* Synchronous execute on device memory with the reference's contract:
 * launches on `stream`, waits for it, and returns SFFT_ERR_DOMAIN if any
 * input value was NaN/Inf (checked through a pinned, mapped per-thread flag:
 * no extra kernel or copy).  If `kernel_ms` is non-NULL it receives the
 * kernel's device time from CUDA events recorded around the launch. */
int sfft_execute_sync(sfft_plan_t plan, const void* d_in, void* d_out, int64_t batch,
                      void* stream, float* kernel_ms);

/* Input kinds of the _ex entry points.  SFFT_INPUT_REAL: `d_in` holds
 * `batch` rows of n REAL values (float for SFFT_SINGLE, double for
 * SFFT_DOUBLE; 16-byte aligned like complex input -- the real loaders read
 * 16-byte chunks of reals) -- the C2C transform of a real signal, as
 * the reference computes for real input (executor.py:74 casts it to
 * complex; tests/test_executor.py:89-92).  The kernel reads the reals and
 * zero imaginary parts in registers: half the input traffic, no widening
 * pass.  Available when sfft_plan_info().real_input is 1 (every default
 * kernel variant); otherwise SFFT_ERR_ARGUMENT. */
#define SFFT_INPUT_COMPLEX 0
#define SFFT_INPUT_REAL 1

/* sfft_execute / sfft_execute_sync with an input kind. */
int sfft_execute_ex(sfft_plan_t plan, const void* d_in, void* d_out, int64_t batch, void* stream,
                    int32_t* d_nonfinite, int32_t input_kind);
int sfft_execute_sync_ex(sfft_plan_t plan, const void* d_in, void* d_out, int64_t batch,
                         void* stream, float* kernel_ms, int32_t input_kind);

/* Synchronous execute on host memory: chunked H2D -> kernel -> D2H pipeline
 * over several streams (pinned memory gives full PCIe/C2C bandwidth);
 * calls of up to 1 MiB of output run zero-copy: one kernel launch reads and
 * writes page-locked, host-mapped memory directly (16-byte aligned pinned
 * user buffers in place, pageable ones through a mapped staging buffer), no
 * copy-engine transfers (SFFT_ZERO_COPY_BYTES=0 restores the single-stream
 * H2D/D2H path for those calls).  The streams, device chunk buffers and
 * pinned staging belong to the device, are shared by all plans on it and
 * live as long as the process; host calls on one device run one at a time.
 * Returns SFFT_ERR_DOMAIN if the input held NaN/Inf (output then undefined). */
int sfft_execute_host(sfft_plan_t plan, const void* h_in, void* h_out, int64_t batch);

/* sfft_execute_host with an input kind: SFFT_INPUT_REAL moves n reals per
 * row host->device (half the H2D bytes) and returns complex rows. */
int sfft_execute_host_ex(sfft_plan_t plan, const void* h_in, void* h_out, int64_t batch,
                         int32_t input_kind);

/* Stage-level API (kernels.py:28-151, planner.py:62-89) on device buffers --
 * not the hot path (that is sfft_execute: all stages fused in one HBM pass),
 * but the reference's building blocks for custom stage lists.
 *
 * sfft_permute: out[r, p] = in[r, perm[p]] for `batch` rows of n elements
 *   (the digit-reversal load of executor.py:77); perm is int64 on device;
 *   an entry outside [0, n) reads nothing and yields NaN in that slot.
 * sfft_stage: one out-of-place radix-2/4/8 decimation-in-time stage over
 *   sub-spectra of length `stride`; operand (q, j) of each group is scaled
 *   by table[(n/(radix*stride))*q*j mod n] (conjugated for SFFT_INVERSE);
 *   `d_table` is the n-entry base table of sfft_build_twiddle_table on the
 *   device.  SFFT_ERR_PLAN if radix*stride does not divide n. */
int sfft_permute(int32_t n, int32_t precision, const int64_t* d_perm, const void* d_in,
                 void* d_out, int64_t batch, void* stream);
int sfft_stage(int32_t n, int32_t precision, int32_t radix, int32_t stride, int32_t direction,
               const void* d_table, const void* d_in, void* d_out, int64_t batch, void* stream);

/* Thread-local message describing the last non-OK status on this thread. */
const char* sfft_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* SFFT_H_ */
