#!/bin/bash
# fiber path with two groups' row loads in flight (PLAIN bit 4096, R = 64 4-mode): tests + benches
o=gpurun_out/r02aa; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "fiber" > $o/fiber_tests.txt 2>&1
for c in cfg3s cfg5s; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $o/bench_$c.json 2> $o/bench_$c.err; done
timeout 1800 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu > $o/bench_cfg5.json 2> $o/bench_cfg5.err
for f in $o/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'], [round(x,2) for x in d['roofline']['kernel_ms_per_mode']], (d.get('parity') or {}).get('ok'))"; done
