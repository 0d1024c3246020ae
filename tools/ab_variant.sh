# A/B two kernel variants (bench --variant) alternating on one box: $1 out dir, $2 A, $3 B
set -x
out=$1; a=$2; b=$3; mkdir -p $out
for i in 1 2; do
  for v in $a $b; do
    python bench.py --variant $v --no-cpu > $out/cfg2_v${v}_$i.json 2>>$out/err.log
    python bench.py --config cfg4s --variant $v --no-cpu > $out/cfg4s_v${v}_$i.json 2>>$out/err.log
  done
done
