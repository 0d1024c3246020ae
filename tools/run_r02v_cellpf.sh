#!/bin/bash
# r02v: per-line prefetch.global.L2 of the blocks cell c+PFD brings in (variants 2-4)
# (historical: variants 2-4 were removed after this sweep; results in
# profiles/sweeps/r02s_cells_wide_negative.jsonl)
o=gpurun_out/r02v; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_cells.py -x -q > $o/cells_tests.txt 2>&1
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0,1 --reps 5 \
  --specs '[{"variant":1},{"variant":2},{"variant":3},{"variant":4}]' > $o/sweep_pf.jsonl 2> $o/sweep_pf.err
