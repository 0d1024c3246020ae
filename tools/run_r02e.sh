#!/bin/bash
# streamed-input cache policy x pinned block size (experiment; SKRP_EXP_STREAM: 0 evict_first, 1 evict_last, 2 no hint)
o=gpurun_out/r02e; mkdir -p $o
for x in 0 1 2; do
  SKRP_EXP_STREAM=$x timeout 900 python tools/sweep_layout.py --config cfg2 --specs tools/sweeps/r02e_stream_policy.json --reps 3 > $o/sweep_stream_$x.jsonl 2> $o/sweep_stream_$x.err
done
