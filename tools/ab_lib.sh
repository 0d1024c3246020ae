# A/B two builds of the library on one box: ab/lib_old.so vs ab/lib_new.so,
# alternating; args: output dir, then bench/sweep command lines via CMDS file
set -x
out=$1; mkdir -p $out
L=paper_2507_15121_b200/libshardkrp_cuda.so
for i in 1 2; do
  for v in old new; do
    cp ab/lib_$v.so $L
    python bench.py --config cfg4s --no-cpu > $out/cfg4s_${v}_$i.json 2>>$out/err.log
    python tools/sweep_layout.py --specs tools/sweeps/specs_2d_ncu.json --reps 3 > $out/sweep2d_${v}_$i.jsonl 2>>$out/err.log
    python bench.py --no-cpu > $out/cfg2_${v}_$i.json 2>>$out/err.log
  done
done
cp ab/lib_new.so $L
