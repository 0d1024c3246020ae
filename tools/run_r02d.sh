#!/bin/bash
# pruned dispatch: full GPU suite, benches (cfg2 default/det, cfg5s, cfg4s, cfg3s, cfg1, reference arm),
# ncu --set full of the new kernel instantiations (summarised on the box)
o=gpurun_out/r02d; mkdir -p $o; t=/tmp/r02d; mkdir -p $t
timeout 1800 python -m pytest tests/ -x -q -m gpu > $o/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu --accumulation deterministic-reduce > $o/bench_cfg2_det.json 2> $o/bench_cfg2_det.err
for c in cfg5s cfg4s cfg3s cfg1; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $o/bench_$c.json 2> $o/bench_$c.err; done
N="ncu --set full --import-source on --clock-control none"
S="python tools/ncu_summary.py full"
timeout 900 $N -k regex:mttkrp_v2 -c 3 -o $t/cfg2_modes python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/ncu_cfg2.log 2>&1
$S $t/cfg2_modes.ncu-rep $o/ncu_cfg2_modes.json --config cfg2 > /dev/null 2>&1
timeout 900 $N -k regex:mttkrp_panel -c 3 -o $t/cfg2_det_modes python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e-api --accumulation deterministic-reduce > $o/ncu_cfg2_det.log 2>&1
$S $t/cfg2_det_modes.ncu-rep $o/ncu_cfg2_det_modes.json --config cfg2 > /dev/null 2>&1
timeout 900 $N -k regex:mttkrp -c 3 -o $t/cfg4s_modes python bench.py --config cfg4s --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/ncu_cfg4s.log 2>&1
$S $t/cfg4s_modes.ncu-rep $o/ncu_cfg4s_modes.json --config cfg4s > /dev/null 2>&1
timeout 900 $N -k regex:mttkrp -c 4 -o $t/cfg5s_modes python bench.py --config cfg5s --steps 3 --warmup 3 --no-cpu --no-parity > $o/ncu_cfg5s.log 2>&1
$S $t/cfg5s_modes.ncu-rep $o/ncu_cfg5s_modes.json --config cfg5s > /dev/null 2>&1
timeout 900 $N -k regex:mttkrp -c 3 -o $t/cfg3s_modes python bench.py --config cfg3s --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/ncu_cfg3s.log 2>&1
$S $t/cfg3s_modes.ncu-rep $o/ncu_cfg3s_modes.json --config cfg3s > /dev/null 2>&1
ncu -i $t/cfg2_modes.ncu-rep --page source --csv 2>/dev/null | gzip -c > $o/cfg2_modes.src.csv.gz
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/launches.log 2>&1
du -sh $o > $o/size.txt
