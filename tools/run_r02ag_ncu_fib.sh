#!/bin/bash
# ncu of the R = 32 fiber kernel with the cp.async metadata ring (cfg3s, 3 modes)
o=gpurun_out/r02ag; mkdir -p $o
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mttkrp_v2 -c 3 -o $o/ncu_cfg3s_smeta python bench.py --config cfg3s --steps 1 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/ncu.log 2>&1
