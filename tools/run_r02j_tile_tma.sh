# tile kernel with the streamed input through a TMA gather4 ring: tests, whole-step A/B, ncu
o=gpurun_out/r02l; mkdir -p $o
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "tma or stream or blocked" > $o/pytest.txt 2>&1
tail -3 $o/pytest.txt
for r in 1 2; do
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e-api --no-parity > $o/bench_base_$r.json 2> $o/bench_base_$r.err
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e-api --tile-tma $( [ $r = 1 ] && echo "" || echo --no-parity ) > $o/bench_tma_$r.json 2> $o/bench_tma_$r.err
done
for f in $o/bench_*.json; do echo $f; python -c "
import json; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['clocks']['sm_mhz'], d['roofline']['kernel_ms_per_mode'], (d.get('parity') or {}).get('ok'), d['roofline']['kernel'][:60])" 2>&1 | tail -2; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:mttkrp_v2_tma -c 3 -o $o/ncu_tma python bench.py --steps 1 --warmup 3 --no-cpu --no-parity --no-e2e-api --tile-tma > $o/ncu.log 2>&1
tail -2 $o/ncu.log
