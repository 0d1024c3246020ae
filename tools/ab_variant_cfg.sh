# A/B two kernel variants on one config, alternating on one box: $1 out dir, $2 config, $3 A, $4 B
set -x
out=$1; c=$2; a=$3; b=$4; mkdir -p $out
for i in 1 2 3; do
  for v in $a $b; do
    python bench.py --config $c --variant $v --no-cpu > $out/${c}_v${v}_$i.json 2>>$out/err.log
  done
done
