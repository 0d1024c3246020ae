#!/bin/bash
# R = 32 fiber path: cp.async metadata ring two batches ahead + two-batch fiber steps (PLAIN bit 8192)
o=gpurun_out/r02ac; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "fiber or tile or parity" > $o/tests.txt 2>&1
for c in cfg3s; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $o/bench_$c.json 2> $o/bench_$c.err; done
timeout 1800 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu > $o/bench_cfg3.json 2> $o/bench_cfg3.err
for f in $o/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'], [round(x,2) for x in d['roofline']['kernel_ms_per_mode']], (d.get('parity') or {}).get('ok'))" 2>&1 | tail -1; done
