# N repeated default bench runs on one box (run-to-run spread of the headline)
out=${1:-gpurun_out/repeat}; n=${2:-5}; mkdir -p $out
for i in $(seq 1 $n); do python bench.py --no-cpu > $out/run_$i.json 2>>$out/err.log; done
