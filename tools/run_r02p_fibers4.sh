# 4-mode fiber layout: tests, cfg5 full / cfg5s
o=gpurun_out/r02p; mkdir -p $o
timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "fiber" > $o/pytest.txt 2>&1
tail -3 $o/pytest.txt
timeout 1800 python bench.py --config cfg5 --steps 3 --warmup 3 --no-cpu > $o/bench_cfg5.json 2> $o/bench_cfg5.err
timeout 900 python bench.py --config cfg5s --steps 5 --warmup 3 --no-cpu > $o/bench_cfg5s.json 2> $o/bench_cfg5s.err
for f in $o/bench_*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_ms_per_mode'], (d.get('parity') or {}).get('ok'), (d.get('parity') or {}).get('max_rel_err'), d['config'].get('layout'))" 2>&1 | tail -2; done
