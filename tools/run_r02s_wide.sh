#!/bin/bash
# r02s (historical): wide cells-kernel variants 2-13 (4 lanes x 32-B rows,
# 8 warps, direct entry loads, register ring, L2 prefetch, flush disabled) were
# instantiated in a working copy of csrc/mttkrp_cells.cu, swept on cfg2 with
# this command and removed after measuring slower than variant 1 -- results in
# profiles/sweeps/r02s_cells_wide_negative.jsonl and
# profiles/r02/r02s_ncu_cells_wide_negative.json.  With the current library only
# variants 0 and 1 exist.
o=gpurun_out/r02s; mkdir -p $o
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0 --reps 5 \
  --specs '[{"variant":1},{"variant":0}]' > $o/sweep.jsonl 2> $o/sweep.err
