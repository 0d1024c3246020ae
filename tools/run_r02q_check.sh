o=gpurun_out/r02q; mkdir -p $o
for c in cfg4s cfg3s cfg1; do timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > $o/bench_$c.json 2> $o/bench_$c.err; done
timeout 900 python bench.py --config cfg4s --steps 5 --warmup 3 --no-cpu --layout flycoo > $o/bench_cfg4s_flycoo.json 2> $o/bench_cfg4s_flycoo.err
for f in $o/bench_*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_ms_per_mode'], (d.get('parity') or {}).get('ok'), d['config'].get('layout'))" 2>&1 | tail -2; done
