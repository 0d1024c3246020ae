set -x
o=gpurun_out/s1; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "slot or invariance_auto" > $o/pytest.txt 2>&1
timeout 900 python bench.py --no-cpu --steps 5 --warmup 3 > $o/bench.json 2> $o/bench.err
timeout 900 python bench.py --no-cpu --steps 5 --warmup 3 --layout blocked > $o/bench_old.json 2> $o/bench_old.err
