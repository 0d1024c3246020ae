# A/B of the run-length output-row ids on cfg2 (alternating runs on one box)
set -x
mkdir -p gpurun_out/rle
python -m pytest tests/test_gpu.py -q -x -k "rle" 2>&1 | tail -3
for i in 1 2; do
  python bench.py --rle-rows 0 --no-cpu > gpurun_out/rle/b0_$i.json 2>>gpurun_out/rle/err.log
  python bench.py --rle-rows 1 --no-cpu > gpurun_out/rle/b1_$i.json 2>>gpurun_out/rle/err.log
done
timeout 600 ncu --set full --clock-control none -k regex:mttkrp_v2 -c 1 -o gpurun_out/rle/v2_rle_mode0 python bench.py --rle-rows 1 --steps 3 --warmup 3 --no-cpu > gpurun_out/rle/ncu.log 2>&1
