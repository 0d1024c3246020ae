#!/bin/bash
# drop-in API with fp32 staging (host-side narrowing / widening): GPU suite + breakdown + bench e2e_api
o=gpurun_out/r02al; mkdir -p $o
timeout 1500 python -m pytest tests/ -q -m gpu > $o/pytest_gpu.txt 2>&1
timeout 900 python tools/profile_e2e_api.py cfg2 > $o/e2e_api.json 2> $o/e2e_api.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --accumulation deterministic-reduce > $o/bench_det.json 2> $o/bench_det.err
python -c "
import json; d=json.loads(open('$o/bench_det.json').read().strip().splitlines()[-1]); print('det', d['ms_per_step'], d['e2e_api'])"
