# After adding the fp64 N=2048 probe variants (LAYOUT 3 split exchange, TWP 3): sanitizers over every
# fp64 N=2048 variant, the full GPU suite, smoke, and a default bench line.
set -x
for tool in racecheck synccheck memcheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_run.py --n 2048 --prec double 2>&1 | tail -2
done
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
python -c "import json; d=json.loads(open('gpurun_out/r02c_bench.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['c4']['gbs'] if 'c4' in d else None)"
