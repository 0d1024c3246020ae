#!/bin/bash
# cells kernel: per-nonzero shared read-add-write (variant 2) vs register runs (variant 1)
# (historical: variant 2 was removed after this sweep)
o=gpurun_out/r02ae; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu_cells.py -x -q > $o/cells_tests.txt 2>&1
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0,1 --reps 3 --specs '[{"variant":1},{"variant":2}]' > $o/sweep.jsonl 2> $o/sweep.err
