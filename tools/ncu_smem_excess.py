"""Per-instruction shared-memory wavefronts from an ncu source page (CSV).

    ncu -i prof.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_smem_excess.py src.csv

Lists every instruction with shared-memory wavefronts (LDS/STS/...) and its
ideal / excessive counts, then the totals -- settles whether bank conflicts
come from the kernel's own accesses or from elsewhere (e.g. bulk-copy writes,
which the per-instruction view does not attribute to an instruction)."""
import csv
import sys


def num(s):
    try:
        return float(str(s).replace(",", ""))
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
hdr = rows[hdr_i]
col = {name: hdr.index(name) for name in hdr}
tot = {"wf": 0.0, "ideal": 0.0, "excess": 0.0}
print(f"{'address':>8} {'wavefronts':>12} {'ideal':>12} {'excessive':>11}  source")
for r in rows[hdr_i + 1:]:
    if len(r) < len(hdr):
        continue
    wf = num(r[col["L1 Wavefronts Shared"]])
    if wf == 0:
        continue
    ideal = num(r[col["L1 Wavefronts Shared Ideal"]])
    exc = num(r[col["L1 Wavefronts Shared Excessive"]])
    tot["wf"] += wf
    tot["ideal"] += ideal
    tot["excess"] += exc
    print(f"{r[col['Address']]:>8} {wf:12.0f} {ideal:12.0f} {exc:11.0f}  {r[col['Source']].strip()[:70]}")
print(f"total instruction-attributed shared wavefronts {tot['wf']:.0f}, ideal {tot['ideal']:.0f}, "
      f"excessive {tot['excess']:.0f} ({100 * tot['excess'] / max(tot['ideal'], 1):.2f} % of ideal)")
