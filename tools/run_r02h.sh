#!/bin/bash
# round-2 final evidence: full GPU suite, bench lines (headline cfg2 with cpu baseline and
# drop-in e2e, deterministic, cells layout, cfg5s/cfg4s/cfg3s/cfg1, reference arm),
# launch list of the headline command, ncu --set full of the cells kernel (all cfg2 modes)
o=gpurun_out/r02h; mkdir -p $o; t=/tmp/r02h; mkdir -p $t
timeout 2400 python -m pytest tests/ -q -m gpu > $o/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --accumulation deterministic-reduce > $o/bench_cfg2_det.json 2> $o/bench_cfg2_det.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --layout cells > $o/bench_cfg2_cells.json 2> $o/bench_cfg2_cells.err
for c in cfg5s cfg4s cfg3s cfg1; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $o/bench_$c.json 2> $o/bench_$c.err; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mttkrp_cells -c 3 -o $t/cells_modes python bench.py --steps 3 --warmup 3 --no-cpu --no-parity --no-e2e-api --layout cells > $o/ncu_cells.log 2>&1
python tools/ncu_summary.py full $t/cells_modes.ncu-rep $o/ncu_cfg2_cells_modes.json --config cfg2 > /dev/null 2>&1
du -sh $o > $o/size.txt
