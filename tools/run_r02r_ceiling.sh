#!/bin/bash
# access-pattern ceiling for the tile kernel (tools/pattern_ceiling.cu)
o=gpurun_out/r02r; mkdir -p $o
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv > $o/smi_before.txt
timeout 600 tools/bin/pattern_ceiling > $o/pattern_ceiling.jsonl 2> $o/pattern_ceiling.err
