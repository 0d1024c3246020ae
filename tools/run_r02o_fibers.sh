# fiber layout: full GPU suite, cfg3s / cfg3 A/B (fibers vs the previous plan order), cfg2 check
o=gpurun_out/r02o; mkdir -p $o
timeout 2400 python -m pytest tests/ -q -m gpu -x > $o/pytest_gpu.txt 2>&1
tail -3 $o/pytest_gpu.txt
timeout 900 python bench.py --config cfg3s --steps 5 --warmup 3 --no-cpu > $o/bench_cfg3s_fibers.json 2> $o/bench_cfg3s_fibers.err
timeout 900 python bench.py --config cfg3s --steps 5 --warmup 3 --no-cpu --layout flycoo > $o/bench_cfg3s_flycoo.json 2> $o/bench_cfg3s_flycoo.err
timeout 1800 python bench.py --config cfg3 --steps 5 --warmup 3 --no-cpu > $o/bench_cfg3_fibers.json 2> $o/bench_cfg3_fibers.err
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu --no-e2e-api > $o/bench_cfg2.json 2> $o/bench_cfg2.err
for f in $o/bench_*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_ms_per_mode'], (d.get('parity') or {}).get('ok'), d['config'].get('layout'), d['roofline']['kernel'][:64])" 2>&1 | tail -2; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_v2 -c 3 -o $o/ncu_cfg3s_fibers python bench.py --config cfg3s --steps 1 --warmup 3 --no-cpu --no-parity --no-e2e-api > $o/ncu.log 2>&1
tail -1 $o/ncu.log
