# A/B two library builds on the deterministic (panel) path, alternating on one box
set -x
out=$1; mkdir -p $out
L=paper_2507_15121_b200/libshardkrp_cuda.so
for i in 1 2; do
  for v in old new; do
    cp ab/lib_$v.so $L
    python bench.py --accumulation deterministic-reduce --no-cpu > $out/cfg2det_${v}_$i.json 2>>$out/err.log
    python bench.py --config cfg3s --accumulation deterministic-reduce --no-cpu > $out/cfg3sdet_${v}_$i.json 2>>$out/err.log
  done
done
cp ab/lib_new.so $L
