set -x
timeout 900 python -m pytest tests/test_gpu_cells.py -x -q 2>&1 | tail -15 > gpurun_out/r2_cells_tests.txt
cat gpurun_out/r2_cells_tests.txt
timeout 1200 python tools/sweep_cells.py --config cfg2 --modes 0,1 --baseline --specs '[{"lag":2},{"lag":0},{"lag":1},{"lag":6},{"lag":2,"flags":1},{"lag":2,"flags":9},{"lag":2,"inner_mb":4},{"lag":2,"inner_mb":16},{"lag":2,"outer_mb":64}]' > gpurun_out/r2_sweep.jsonl 2> gpurun_out/r2_sweep.err
cat gpurun_out/r2_sweep.jsonl | cut -c1-220; tail -5 gpurun_out/r2_sweep.err
timeout 600 ncu --set full --import-source on -k regex:mttkrp_cells -c 1 -o gpurun_out/r2_ncu_cells_mode0 python tools/sweep_cells.py --config cfg2 --modes 0 --reps 1 --specs '[{"lag":2}]' > gpurun_out/r2_ncu.log 2>&1
tail -5 gpurun_out/r2_ncu.log
