#!/bin/bash
# cells kernel: warp-uniform skip of the flush (variant 2) x cell sizes
# (historical: variant 2 was removed after this sweep; results in
# profiles/sweeps/r02s_cells_wide_negative.jsonl)
o=gpurun_out/r02z; mkdir -p $o
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0 --reps 3 \
  --specs '[{"variant":1},{"variant":2},{"variant":1,"inner_mb":32},{"variant":2,"inner_mb":32},{"variant":2,"inner_mb":32,"outer_mb":64},{"variant":2,"inner_mb":64,"outer_mb":32},{"variant":1,"inner_mb":64,"outer_mb":64},{"variant":2,"inner_mb":64,"outer_mb":64}]' > $o/sweep.jsonl 2> $o/sweep.err
