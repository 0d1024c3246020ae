set -x
timeout 900 python -m pytest tests/test_gpu_cells.py -x -q 2>&1 | tail -25 > gpurun_out/r8_cells_tests.txt
cat gpurun_out/r8_cells_tests.txt
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0,1 --baseline --specs '[{"lag":2},{"lag":0},{"lag":4},{"lag":2,"inner_mb":16},{"lag":2,"inner_mb":4},{"lag":8}]' > gpurun_out/r8_sweep.jsonl 2> gpurun_out/r8_sweep.err
cut -c1-200 gpurun_out/r8_sweep.jsonl; tail -3 gpurun_out/r8_sweep.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_cells -c 1 -o gpurun_out/r8_ncu_cells_mode0 python tools/sweep_cells.py --config cfg2 --modes 0 --reps 1 --specs '[{"lag":2}]' > gpurun_out/r8_ncu.log 2>&1
tail -3 gpurun_out/r8_ncu.log
