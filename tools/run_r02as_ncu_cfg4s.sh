#!/bin/bash
# ncu of the cfg4s (Zipf) tile-kernel launches: what bounds the Zipf configs
o=gpurun_out/r02as; mkdir -p $o
timeout 900 ncu --set full --clock-control none -k regex:mttkrp_v2 -c 3 -o $o/ncu_cfg4s python bench.py --config cfg4s --steps 1 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/ncu.log 2>&1
