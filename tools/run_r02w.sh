#!/bin/bash
# bench line with roofline.frac_miss_pattern (cfg2) + ncu of the cfg5s kernels (what bounds CP-ALS)
o=gpurun_out/r02w; mkdir -p $o
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 900 ncu --set full --clock-control none -k regex:mttkrp_v2 -c 4 -o $o/ncu_cfg5s python bench.py --config cfg5s --steps 1 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/ncu.log 2>&1
