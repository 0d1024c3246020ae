#!/bin/bash
# replay the real cells layout without the reduction (tools/replay_cells.cu)
mkdir -p gpurun_out/r02y
timeout 1200 python tools/replay_cells.py --config cfg2 --mode 0 > gpurun_out/r02y/replay.jsonl 2> gpurun_out/r02y/replay.err
