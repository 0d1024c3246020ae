#!/bin/bash
# ncu --set full of the dominant kernel, all three cfg2 modes (default layout), the slot kernel (mode 0),
# cfg4s / cfg5s main kernels; plus the fixed 2-rank test
o=gpurun_out/r02b; mkdir -p $o
free -g > $o/free.txt; nproc > $o/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $o/nproc.txt
timeout 600 python -m pytest tests/test_gpu_dist.py -x -q > $o/pytest_dist.txt 2>&1
N="ncu --set full --import-source on --clock-control none"
timeout 900 $N -k regex:mttkrp_v2 -c 3 -o $o/cfg2_v2_modes python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > $o/ncu_cfg2.log 2>&1
timeout 900 $N -k regex:mttkrp_slots -c 1 -o $o/cfg2_slots_mode0 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --layout slots > $o/ncu_slots.log 2>&1
timeout 900 $N -k regex:mttkrp -c 3 -o $o/cfg4s_modes python bench.py --config cfg4s --steps 3 --warmup 3 --no-cpu --no-parity > $o/ncu_cfg4s.log 2>&1
timeout 900 $N -k regex:mttkrp -c 4 -o $o/cfg5s_modes python bench.py --config cfg5s --steps 3 --warmup 3 --no-cpu --no-parity > $o/ncu_cfg5s.log 2>&1
