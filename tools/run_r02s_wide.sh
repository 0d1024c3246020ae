#!/bin/bash
o=gpurun_out/r02s; mkdir -p $o
timeout 1500 python tools/sweep_cells.py --config cfg2 --modes 0 --reps 5 \
  --specs '[{"variant":1},{"variant":11},{"variant":12}]' > $o/sweep_pf.jsonl 2> $o/sweep_pf.err
