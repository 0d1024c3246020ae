#!/bin/bash
# packed-metadata tile kernel A/B on cfg2 (tools/packed_probe.py) + ncu of both kernels (mode 0)
# HISTORICAL: the packed-metadata kernel (SKRP_FLAG_PACKED, PLAIN bit 32768) was
# removed after this A/B (profiles/sweeps/r02an_packed_metadata_negative.jsonl);
# this script and tools/historical/packed_probe.py no longer run against the library.
o=gpurun_out/r02an; mkdir -p $o
timeout 1500 python tools/packed_probe.py --modes 0,1,2 --reps 5 > $o/probe.jsonl 2> $o/probe.err
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:mttkrp_v2 --launch-skip 1 --launch-count 1 -c 1 --csv --log-file $o/ncu_prod.csv python tools/packed_probe.py --modes 0 --reps 1 > $o/ncu_prod.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:mttkrp_v2 --launch-skip 2 --launch-count 1 --csv --log-file $o/ncu_packed.csv python tools/packed_probe.py --modes 0 --reps 1 > $o/ncu_packed.log 2>&1
