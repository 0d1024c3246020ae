# full-size cfg5 (4-mode 2B-nnz Zipf, R=64, one CP-ALS iteration) on ONE B200: plans built
# in their execution layout and parked on the host while the next mode sorts
o=gpurun_out/r02m; mkdir -p $o
(while true; do nvidia-smi --query-gpu=memory.used,memory.total --format=csv,noheader >> $o/mem_trace.txt; free -g | awk '/Mem/{print "host", $3, $7}' >> $o/mem_trace.txt; sleep 5; done) &
MON=$!
timeout 1800 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu --accumulation deterministic-reduce > $o/bench_cfg5_det.json 2> $o/bench_cfg5_det.err
echo "rc=$?" >> $o/bench_cfg5_det.err
kill $MON
tail -3 $o/bench_cfg5_det.err
