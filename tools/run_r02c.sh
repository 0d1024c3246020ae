#!/bin/bash
# ncu --set full of the mttkrp kernels (summarised ON the box: reports are too big to bring back),
# the new scale tests, the fixed 2-rank test, bench cfg2 + cfg5s with the new parity blocks
o=gpurun_out/r02c; mkdir -p $o; t=/tmp/r02c; mkdir -p $t
free -g > $o/free.txt; nproc > $o/nproc.txt; grep -m1 "model name" /proc/cpuinfo >> $o/nproc.txt
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_scale.py -x -q > $o/pytest_dist_scale.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 900 python bench.py --config cfg5s --steps 3 --warmup 3 --no-cpu > $o/bench_cfg5s.json 2> $o/bench_cfg5s.err
N="ncu --set full --import-source on --clock-control none"
S="python tools/ncu_summary.py full"
timeout 900 $N -k regex:mttkrp_v2 -c 3 -o $t/cfg2_v2_modes python bench.py --steps 3 --warmup 3 --no-cpu --no-parity > $o/ncu_cfg2.log 2>&1
$S $t/cfg2_v2_modes.ncu-rep $o/ncu_cfg2_v2_modes.json --config cfg2 > /dev/null 2>&1
timeout 900 $N -k regex:mttkrp_slots -c 1 -o $t/cfg2_slots_mode0 python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --layout slots > $o/ncu_slots.log 2>&1
$S $t/cfg2_slots_mode0.ncu-rep $o/ncu_cfg2_slots_mode0.json --config cfg2 > /dev/null 2>&1
timeout 900 $N -k regex:mttkrp -c 3 -o $t/cfg4s_modes python bench.py --config cfg4s --steps 3 --warmup 3 --no-cpu --no-parity > $o/ncu_cfg4s.log 2>&1
$S $t/cfg4s_modes.ncu-rep $o/ncu_cfg4s_modes.json --config cfg4s > /dev/null 2>&1
timeout 900 $N -k regex:mttkrp -c 4 -o $t/cfg5s_modes python bench.py --config cfg5s --steps 3 --warmup 3 --no-cpu --no-parity > $o/ncu_cfg5s.log 2>&1
$S $t/cfg5s_modes.ncu-rep $o/ncu_cfg5s_modes.json --config cfg5s > /dev/null 2>&1
ls -la $t > $o/reps.txt
for f in cfg2_v2_modes cfg2_slots_mode0; do ncu -i $t/$f.ncu-rep --page source --csv > $t/$f.src.csv 2>/dev/null; gzip -c $t/$f.src.csv > $o/$f.src.csv.gz; done
du -sh $o >> $o/reps.txt
