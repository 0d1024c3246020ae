# A/B on one box: default (tile kernel) vs cells layout, whole bench steps (power-capped regime)
o=gpurun_out/r14; mkdir -p $o
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e-api > $o/bench_default.json 2> $o/bench_default.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e-api --layout cells > $o/bench_cells.json 2> $o/bench_cells.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e-api --no-parity > $o/bench_default2.json 2> $o/bench_default2.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e-api --no-parity --layout cells > $o/bench_cells2.json 2> $o/bench_cells2.err
for f in $o/*.json; do echo $f; python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks'], d['roofline']['kernel_ms_per_mode'] if 'kernel_ms_per_mode' in d.get('roofline',{}) else '', (d.get('parity') or {}).get('ok'))"; done
