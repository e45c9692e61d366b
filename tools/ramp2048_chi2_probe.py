"""Why does the reference's frozen chi2 == 0 check (tests/test_stats.py:211-222)
fail on the GPU engine?  Compares each pair of {GPU engine, reference-formula
naive DFT (numpy), package naive_dft (GPU)} for ramp-2048."""
import numpy as np

import oracle as ora
import paper_2203_09384_b200 as sf
from paper_2203_09384_b200.stats import compare_spectra

x = sf.generate("ramp", 2048)
engine = sf.execute(sf.make_plan(2048), x)
ref_engine = ora.reference_execute(x[None], "forward", dtype=np.complex64)[0]
k = np.arange(2048)
m = np.exp((-2.0j * np.pi / 2048) * (np.outer(k, k) % 2048))
ref_naive = (m @ x.astype(np.complex128)).astype(np.complex64)
gpu_naive = sf.naive_dft(x)
for a, b, name in [(engine, ref_naive, "engine vs numpy naive"), (engine, gpu_naive, "engine vs gpu naive"),
                   (ref_engine, ref_naive, "ref engine vs numpy naive"), (gpu_naive, ref_naive, "gpu naive vs numpy naive"),
                   (engine, ref_engine, "engine vs ref engine")]:
    r = compare_spectra(a, b)
    print(f"{name:28s} chi2={r.chi2_reduced:.3e} p={r.p_value:.6f} maxrel={r.max_rel_diff:.2e} "
          f"absmax={r.abs_diff_max:.3e} ne={int(np.sum(a != b))}")
va, vb = np.abs(engine).astype(np.float64), np.abs(ref_naive).astype(np.float64)
lo, hi = min(va.min(), vb.min()), max(va.max(), vb.max())
e = np.linspace(lo, hi, 2049)
ia, ib = np.searchsorted(e, va, side="right") - 1, np.searchsorted(e, vb, side="right") - 1
for i in np.flatnonzero(ia != ib):
    print("bin flip at k=", i, va[i], vb[i], "edge", e[max(ia[i], ib[i])])

# per-variant ramp abs error (reference test bound: abs_diff_max < 0.1) and random rel-L2
lib = sf._native.lib()
xr = sf.generate_batch(256, 2048, seed=1)
exact_r = ora.direct_dft(xr)
for prec in ("single",):
    for v in range(lib.sfft_num_variants(2048, 0)):
        p = sf.make_plan(2048, variant=v)
        info = p.kernel_info(0)
        y = sf.execute(p, x)
        yr = sf.execute(p, xr)
        rel = np.max(np.linalg.norm(yr - exact_r, axis=1) / np.linalg.norm(exact_r, axis=1))
        print(f"v{v} R={info['elems_per_thread']} twp={info['twiddle_policy']} layout={info['layout']} "
              f"ramp absmax={np.abs(y.astype(np.complex128) - ref_naive).max():.4f} random relL2max={rel:.3e}")
