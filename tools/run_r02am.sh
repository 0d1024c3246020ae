#!/bin/bash
# round-2 final evidence (final code: fiber metadata ring, fp32-staged drop-in I/O): GPU suite, bench lines, launch list
o=gpurun_out/r02am; mkdir -p $o
timeout 2400 python -m pytest tests/ -q -m gpu > $o/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $o/bench_reference.json 2> $o/bench_reference.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --accumulation deterministic-reduce > $o/bench_cfg2_det.json 2> $o/bench_cfg2_det.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --layout cells > $o/bench_cfg2_cells.json 2> $o/bench_cfg2_cells.err
for c in cfg5s cfg4s cfg3s cfg1; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $o/bench_$c.json 2> $o/bench_$c.err; done
timeout 1800 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu > $o/bench_cfg5.json 2> $o/bench_cfg5.err
timeout 1800 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu > $o/bench_cfg3.json 2> $o/bench_cfg3.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/launches.log 2>&1
du -sh $o > $o/size.txt
