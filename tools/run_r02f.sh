#!/bin/bash
# full GPU suite, cfg2 / cfg5s lines with the ncu traffic table, full-size cfg3 on one GPU (host-memory watchdog)
o=gpurun_out/r02f; mkdir -p $o
timeout 1800 python -m pytest tests/ -q -m gpu > $o/pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > $o/bench_cfg2.json 2> $o/bench_cfg2.err
timeout 900 python bench.py --config cfg5s --steps 5 --warmup 3 --no-cpu > $o/bench_cfg5s.json 2> $o/bench_cfg5s.err
# cfg3 full: 3.6e9 nnz; kill it if host memory runs low (the parked plans live in host RAM)
timeout 1500 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu > $o/bench_cfg3.json 2> $o/bench_cfg3.err &
pid=$!
while kill -0 $pid 2>/dev/null; do
  avail=$(awk '/MemAvailable/ {print $2}' /proc/meminfo)
  echo "$(date +%s) $avail $(nvidia-smi --query-gpu=memory.used --format=csv,noheader,nounits)" >> $o/mem_cfg3.txt
  if [ "$avail" -lt 12000000 ]; then echo "low host memory: killing $pid" >> $o/mem_cfg3.txt; kill -9 $pid; fi
  sleep 2
done
wait $pid; echo "cfg3 rc=$?" >> $o/mem_cfg3.txt
