set -x
timeout 900 python -m pytest tests/test_gpu_cells.py -x -q 2>&1 | tail -3 > gpurun_out/r17_cells_tests.txt
cat gpurun_out/r17_cells_tests.txt
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0,1 --baseline --specs '[{"variant":1},{"variant":1,"lag":2},{"variant":0}]' > gpurun_out/r17_sweep.jsonl 2> gpurun_out/r17_sweep.err
cut -c1-160 gpurun_out/r17_sweep.jsonl; tail -3 gpurun_out/r17_sweep.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_cells -c 1 -o gpurun_out/r17_ncu_cells_mode0 python tools/sweep_cells.py --config cfg2 --modes 0 --reps 1 --specs '[{"variant":1}]' > gpurun_out/r17_ncu.log 2>&1
tail -2 gpurun_out/r17_ncu.log
