"""SASS evidence for the shipped library: per-kernel instruction counts.

Runs ``cuobjdump -sass`` on ``paper_2203_09384_b200/_lib/libsfft.so`` (all
sm_100a cubins) and counts, per kernel, the instructions that show the
Blackwell-native code paths:

* bulk TMA + mbarrier: ``UBLKCP`` (cp.async.bulk), ``SYNCS.*`` (mbarrier ops);
* packed FP32x2 pipe: ``FADD2`` / ``FMUL2`` / ``FFMA2``; scalar FP64:
  ``DADD`` / ``DMUL`` / ``DFMA``;
* global and shared access widths: ``LDG``/``STG``/``LDS``/``STS`` by width
  (32 / 64 / 128 bit), ``LDGSTS`` (cp.async), ``BAR``;
* tensor memory: ``UTCCP`` (tcgen05.cp smem -> TMEM), ``LDTM`` (tcgen05.ld);
* total static instruction count.

Default kernels (variant 0 of each length / precision / direction / input
kind, as ``sfft_variant_info`` reports them) are marked.  Static counts: a
kernel's body is fully unrolled, so they are per thread per CTA lifetime.

    python tools/sass_summary.py [--all] [--json out.json] > profiles/r02_sass_summary.txt
"""
import argparse
import collections
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2203_09384_b200", "_lib", "libsfft.so")

OPS = ("UBLKCP", "SYNCS", "FADD2", "FMUL2", "FFMA2", "FADD", "FMUL", "FFMA", "DADD", "DMUL", "DFMA", "LDGSTS",
       "BAR", "SHFL", "UTCCP", "LDTM")


def demangle(names):
    out = subprocess.run(["cu++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return dict(zip(names, out))


def width(mnemonic: str) -> str:
    m = re.search(r"\.(64|128)\b", mnemonic)
    return m.group(1) if m else "32"


def parse(sass: str):
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if not m:
            continue
        mnem = m.group(2)
        base = mnem.split(".")[0]
        c = kernels[cur]
        c["total"] += 1
        if base in ("LDG", "STG", "LDS", "STS"):
            c[f"{base}.{width(mnem)}"] += 1
        elif base in OPS:
            c[base] += 1
        elif base.startswith("SYNCS"):
            c["SYNCS"] += 1
    return kernels


def default_signatures():
    """(precision letter, N, R, SEQ, LAYOUT, TWP, LOADER) of every default Stockham variant and
    (precision letter, N, SPT?, ...) of tile defaults, from the native variant table."""
    import paper_2203_09384_b200 as sf

    sigs = set()
    for prec, code, letter in (("single", 0, "f"), ("double", 1, "d")):
        for p in range(1, 12):
            n = 2**p
            info = sf._native.variant_info(n, code, 0)
            if info["kernel"] == sf._native.SFFT_KERNEL_STOCKHAM:
                sigs.add(("stockham", letter, n, info["elems_per_thread"], info["seqs_per_cta"], info["layout"],
                          info["twiddle_policy"], info["loader"]))
            else:
                sigs.add(("tile", letter, n, info["seqs_per_cta"], info["threads_per_cta"]))
    return sigs


def classify(demangled: str, sigs):
    d = re.sub(r"\((?:int|bool)\)", "", demangled)  # cu++filt spells template args as (int)1024, (bool)0
    m = re.search(r"sfft::stockham_kernel(?:_capped)?<(float|double), (\d+), (\d+), (\d+), ([01]), (\d), (\d), (\d), "
                  r"([01])(?:, (\d+))?>", d)
    if m:
        letter = "f" if m.group(1) == "float" else "d"
        key = ("stockham", letter, int(m.group(2)), int(m.group(3)), int(m.group(4)), int(m.group(6)),
               int(m.group(7)), int(m.group(8)))
        label = (f"stockham {m.group(1)} N={m.group(2)} R={m.group(3)} seq={m.group(4)} "
                 f"{'inv' if m.group(5) == '1' else 'fwd'} layout={m.group(6)} twp={m.group(7)} "
                 f"loader={m.group(8)}{' real-in' if m.group(9) == '1' else ''}"
                 f"{' minb=' + m.group(10) if m.group(10) else ''}")
        return label, key in sigs
    m = re.search(r"sfft::tile_kernel<(float|double), (\d+), (\d+), (\d+), ([01]), ([01])>", d)
    if m:
        letter = "f" if m.group(1) == "float" else "d"
        spt, warps = int(m.group(3)), int(m.group(4))
        key = ("tile", letter, int(m.group(2)), 32 * spt * warps, 32 * warps)
        label = (f"tile {m.group(1)} N={m.group(2)} spt={spt} warps={warps} "
                 f"{'inv' if m.group(5) == '1' else 'fwd'}{' real-in' if m.group(6) == '1' else ''}")
        return label, key in sigs
    m = re.search(r"sfft::split2_kernel<(float|double), (\d+), (\d+), ([01]), (\d), (\d), ([01])>", d)
    if m:
        return (f"split2 {m.group(1)} N={m.group(2)} R={m.group(3)} {'inv' if m.group(4) == '1' else 'fwd'} "
                f"layout={m.group(5)} twp={m.group(6)}{' real-in' if m.group(7) == '1' else ''}"), False
    m = re.search(r"sfft::stockham_tmem_kernel<(float|double), (\d+), (\d+), ([01]), (\d), ([01]), (\d), ([01])>", d)
    if m:
        return (f"stockham_tmem {m.group(1)} N={m.group(2)} R={m.group(3)} {'inv' if m.group(4) == '1' else 'fwd'} "
                f"twp={m.group(5)} minb={m.group(7)} loader={'3' if m.group(8) == '1' else '4'}"
                f"{' real-in' if m.group(6) == '1' else ''}"), False
    m = re.search(r"sfft::fourstep_kernel<(float|double), ([01]), ([01]), (\d)>", d)
    if m:
        return (f"fourstep {m.group(1)} N=2048 {'inv' if m.group(2) == '1' else 'fwd'} minb={m.group(4)}"
                f"{' real-in' if m.group(3) == '1' else ''}"), False
    m = re.search(r"sfft::stockham_pipe_kernel<(float|double), (\d+), (\d+), (\d+), ([01])", d)
    if m:
        return (f"stockham_pipe {m.group(1)} N={m.group(2)} R={m.group(3)} seq={m.group(4)} "
                f"{'inv' if m.group(5) == '1' else 'fwd'}"), False
    return demangled.split("(")[0], False


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--all", action="store_true", help="every kernel, not only the defaults")
    ap.add_argument("--json")
    args = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    kernels = parse(sass)
    names = demangle(list(kernels))
    sigs = default_signatures()
    cols = ["total", "UBLKCP", "SYNCS", "FFMA2", "FADD2", "FMUL2", "FFMA", "FADD", "FMUL", "DADD", "DMUL", "DFMA",
            "LDG.32", "LDG.64", "LDG.128", "LDGSTS", "STG.32", "STG.64", "STG.128", "LDS.64", "LDS.128", "STS.64",
            "STS.128", "BAR", "UTCCP", "LDTM"]
    rows = []
    for mangled, c in kernels.items():
        label, is_default = classify(names[mangled], sigs)
        if not (args.all or is_default):
            continue
        rows.append({"kernel": label, "default": is_default, **{k: c.get(k, 0) for k in cols}})
    rows.sort(key=lambda r: r["kernel"])
    print(f"cuobjdump -sass {os.path.relpath(LIB, ROOT)}: {len(kernels)} kernels, all sm_100a; "
          f"{sum(r['default'] for r in rows)} default instantiations listed")
    print("static per-thread instruction counts (fully unrolled bodies)")
    print("kernel".ljust(70) + " ".join(k.rjust(7) for k in cols))
    for r in rows:
        print(r["kernel"].ljust(70) + " ".join(str(r[k]).rjust(7) for k in cols))
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
