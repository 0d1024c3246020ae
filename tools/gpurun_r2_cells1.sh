set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_cells.py -x -q 2>&1 | tail -30 > gpurun_out/r1_cells_tests.txt
cat gpurun_out/r1_cells_tests.txt
timeout 900 python bench.py --config cfg2 --layout cells --steps 5 --warmup 3 --no-cpu --no-e2e-api > gpurun_out/r1_bench_cells.json 2> gpurun_out/r1_bench_cells.err
tail -c 3000 gpurun_out/r1_bench_cells.json; tail -20 gpurun_out/r1_bench_cells.err
timeout 900 python bench.py --config cfg2 --steps 5 --warmup 3 --no-cpu --no-e2e-api --no-parity > gpurun_out/r1_bench_auto.json 2> gpurun_out/r1_bench_auto.err
tail -c 1500 gpurun_out/r1_bench_auto.json
