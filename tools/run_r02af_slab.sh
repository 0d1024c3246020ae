#!/bin/bash
# deterministic-reduce (panel kernel) slab size: 64 KB (512 rows) vs 128 KB (1024 rows)
# result: 64/96 KB 139.8-140.0 ms/step, 128 KB 255 ms (K1b)
o=gpurun_out/r02af; mkdir -p $o
for kb in 64 128 96; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e-api --accumulation deterministic-reduce --panel-smem-kb $kb > $o/bench_det_$kb.json 2> $o/bench_det_$kb.err; done
for f in $o/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'], [round(x,2) for x in d['roofline']['kernel_ms_per_mode']], (d.get('parity') or {}).get('ok'))" 2>&1 | tail -1; done
