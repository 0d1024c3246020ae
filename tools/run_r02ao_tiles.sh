#!/bin/bash
# cfg2 tile-size sweep on the final code (auto = 4096)
o=gpurun_out/r02ao; mkdir -p $o
for t in 4096 2048 8192 16384 4096; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e-api --no-parity --tile $t > $o/bench_tile_$t.json 2> $o/bench_tile_$t.err; python -c "
import json; d=json.loads(open('$o/bench_tile_$t.json').read().strip().splitlines()[-1]); print($t, d['ms_per_step'], d['clocks']['sm_mhz'], [round(x,2) for x in d['roofline']['kernel_ms_per_mode']])"; done
