#!/bin/bash
# A/B on one box: cfg2 with the metadata ring in the pin-one-stream-one kernel (smeta) vs production
# (historical: the smeta build was a working-copy variant, not kept; results in
# profiles/sweeps/r02ap_cfg2_metadata_ring_negative.jsonl)
o=gpurun_out/r02ap; mkdir -p $o
L=paper_2507_15121_b200
for v in prod smeta prod smeta; do
  cp $L/libshardkrp_cuda_${v}_ab.so $L/libshardkrp_cuda.so
  timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e-api > $o/bench_$v.json 2> $o/bench_$v.err
  python -c "
import json; d=json.loads(open('$o/bench_$v.json').read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['clocks']['sm_mhz'], [round(x,2) for x in d['roofline']['kernel_ms_per_mode']], d['roofline']['per_mode'][0]['kernel'], (d.get('parity') or {}).get('ok'))"
done
cp $L/libshardkrp_cuda_smeta_ab.so $L/libshardkrp_cuda.so
