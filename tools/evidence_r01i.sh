set -x
mkdir -p gpurun_out/r01i
python bench.py > gpurun_out/r01i/bench_default.json 2> gpurun_out/r01i/bench_default.err
python bench.py --impl reference > gpurun_out/r01i/bench_reference.json 2> gpurun_out/r01i/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01i/launches.csv python bench.py --steps 3 --warmup 3 > gpurun_out/r01i/launches_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:mttkrp_v2 -c 1 -o gpurun_out/r01i/v2_mode0 python bench.py --steps 3 --warmup 3 > gpurun_out/r01i/full.log 2>&1
python bench.py --accumulation deterministic-reduce > gpurun_out/r01i/bench_det.json 2> gpurun_out/r01i/bench_det.err
