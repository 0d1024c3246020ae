#!/bin/bash
# R = 64 general path: class-0 batches issue two groups' row loads (PLAIN bit 16384)
# (historical: PLAIN bit 16384 was removed after this measurement)
o=gpurun_out/r02ad; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "fiber or tile or parity or cpd or four" > $o/tests.txt 2>&1
timeout 900 python bench.py --config cfg5s --steps 5 --warmup 3 --no-cpu > $o/bench_cfg5s.json 2> $o/bench_cfg5s.err
timeout 1800 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu > $o/bench_cfg5.json 2> $o/bench_cfg5.err
for f in $o/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'], [round(x,2) for x in d['roofline']['kernel_ms_per_mode']], (d.get('parity') or {}).get('ok'))" 2>&1 | tail -1; done
