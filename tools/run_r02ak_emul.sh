#!/bin/bash
# single-GPU emulation of one rank's share at N = 2/4/8 (projection, not a multi-GPU measurement)
o=gpurun_out/r02ak; mkdir -p $o
for n in 2 4 8; do timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e-api --emulate-world $n > $o/bench_emul_$n.json 2> $o/bench_emul_$n.err; done
for f in $o/bench_*.json; do python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['clocks']['sm_mhz'], d.get('emulated'), (d.get('parity') or {}).get('ok'))" 2>&1 | tail -1; done
