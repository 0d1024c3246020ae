# A/B the panel kernel's per-group CTA barrier on the deterministic cfg2 path (one box, alternating)
set -x
out=$1; mkdir -p $out
for i in 1 2; do
  for v in 0 1; do
    python bench.py --accumulation deterministic-reduce --panel-group-sync $v --no-cpu > $out/det_gs${v}_$i.json 2>>$out/err.log
  done
done
