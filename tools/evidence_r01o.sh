# Round-1 final evidence (after the predicated class-1 FFMAs) for the current kernels (one box, sequential)
set -x
o=gpurun_out/r01o; mkdir -p $o
python bench.py > $o/bench_default.json 2> $o/err.log
python bench.py --impl reference > $o/bench_reference.json 2>> $o/err.log
python bench.py --accumulation deterministic-reduce --no-cpu > $o/bench_det.json 2>> $o/err.log
for c in cfg1 cfg3s cfg4s cfg5s; do python bench.py --config $c --no-cpu > $o/bench_$c.json 2>> $o/err.log; done
for n in 2 4 8; do python bench.py --emulate-world $n --no-cpu > $o/emulated_$n.json 2>> $o/err.log; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $o/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu > $o/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mttkrp_v2 -c 1 -o $o/v2_mode0 python bench.py --steps 3 --warmup 3 --no-cpu > $o/full.log 2>&1
python bench.py > $o/bench_default_run2.json 2>> $o/err.log
