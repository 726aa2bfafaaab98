# Round-2 final refresh (GPU box, repo root): sweep, shard model, launch list of the final code.
set -x
O=gpurun_out
out=$O/sweep_r02c.jsonl; : > $out
for N in 64 128 256 1024 4096 16384; do
  timeout 900 python bench.py --config C5 --members $N --steps 3 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
for C in C1 C2; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
timeout 1200 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c4_r02c.log 2>&1
python tools/shard_model.py --config C3 --graph > $O/shard_model_c3_r02c.log 2>&1
B1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$B1 > $O/b1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3_h50_r02c.csv $B1 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c3_h50_r02c.csv 3 > $O/launches_c3_h50_r02c_summary.txt
