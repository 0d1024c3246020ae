set -x
timeout 900 python -m pytest tests/test_gpu_cells.py -x -q 2>&1 | tail -3 > gpurun_out/r16_cells_tests.txt
cat gpurun_out/r16_cells_tests.txt
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0,1 --baseline --specs '[{"prefetch":false},{"prefetch":true},{"prefetch":true,"lag":2},{"prefetch":false}]' > gpurun_out/r16_sweep.jsonl 2> gpurun_out/r16_sweep.err
cut -c1-160 gpurun_out/r16_sweep.jsonl; tail -3 gpurun_out/r16_sweep.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_cells -c 1 -o gpurun_out/r16_ncu_cells_mode0 python tools/sweep_cells.py --config cfg2 --modes 0 --reps 1 --specs '[{"prefetch":true}]' > gpurun_out/r16_ncu.log 2>&1
tail -2 gpurun_out/r16_ncu.log
