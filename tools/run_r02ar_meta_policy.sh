#!/bin/bash
# A/B on one box: metadata loads L2::evict_normal (slot "smeta") vs evict_first (production)
# (historical: the variant build was a working-copy change, not kept; results in
# profiles/sweeps/r02ar_metadata_policy_negative.jsonl)
o=gpurun_out/r02ar; mkdir -p $o
L=paper_2507_15121_b200
for v in prod smeta prod smeta; do  # smeta slot = metadata evict_normal build
  cp $L/libshardkrp_cuda_${v}_ab.so $L/libshardkrp_cuda.so
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e-api > $o/bench_$v.json 2> $o/bench_$v.err
  python -c "
import json; d=json.loads(open('$o/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['clocks']['sm_mhz'], [round(x,2) for x in d['roofline']['kernel_ms_per_mode']], d['roofline']['per_mode'][0]['kernel'], (d.get('parity') or {}).get('ok'))"
done
cp $L/libshardkrp_cuda_smeta_ab.so $L/libshardkrp_cuda.so
