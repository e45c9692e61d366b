# Large host calls on pinned buffers: zero-copy kernel (SFFT_ZERO_COPY_PINNED=1, an experimental path since removed)
# vs the copy-engine pipeline, c2 e2e.  Result: 13.8 vs 11.9 ms per step -- copy engines win for large calls.
set -x
for i in 1 2; do
  for z in 0 1; do
    SFFT_ZERO_COPY_PINNED=$z python bench.py --steps 10 --warmup 3 --no-cpu --no-extras --e2e-steps 10 > gpurun_out/zcp_$z.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/zcp_$z.json').read().strip().splitlines()[-1]); e=d['e2e']; print('ZC_PINNED=$z', e['value'], e['ms_per_step'], e['link'], e['step_ms_min_median_max'], d['value'])"
  done
done
