# Round-2 profile refresh after the CNN / issuer rework (GPU box, repo root).  Outputs under
# gpurun_out/, summaries copied into profiles/r02/ by hand.  Each ncu command runs only after the
# same program exited 0 without ncu.
set -x
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu_r02b.log 2>&1; tail -2 $O/pytest_gpu_r02b.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02b.log 2>&1
for r in 1 2; do python bench.py > $O/bench_c3_r02b_$r.json 2> $O/bench_c3_r02b_$r.err; done
out=$O/sweep_r02b.jsonl; : > $out
for N in 64 128 256 1024 4096 16384; do
  timeout 900 python bench.py --config C5 --members $N --steps 3 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
for C in C1 C2; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
timeout 1200 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c4_r02b.log 2>&1
python tools/shard_model.py --config C3 --graph > $O/shard_model_c3_r02b.log 2>&1
B1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$B1 > $O/b1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3_h50_r02b.csv $B1 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c3_h50_r02b.csv 1 > $O/launches_c3_h50_r02b_summary.txt
B8="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --horizon 8"
for k in cnn3_tc f16p_gemm_pair noise_kernel center_f16pair_t; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 6 -c 1 \
    -o $O/ncu_r02b_$k $B8 > $O/ncu_r02b_$k.log 2>&1
  python tools/ncu_summary.py $O/ncu_r02b_$k.ncu-rep > $O/ncu_r02b_${k}_summary.txt 2>&1
done
