# Round profile refresh: default bench line, H=50 launch list, ncu --set full of the top kernels,
# config sweep (eager and CUDA-graph).  Run on the GPU box from the repo root.
set -x
python bench.py > gpurun_out/bench_c3.log 2>&1; tail -1 gpurun_out/bench_c3.log > gpurun_out/bench_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_h50.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches_h50.csv 1 > gpurun_out/launches_h50_summary.txt
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --horizon 8"
for k in noise_kernel cnn3_tc center_f16pair_v4 center_f16pair_t f16p_gemm_pair; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 6 -c 1 -o gpurun_out/ncu_$k $B > gpurun_out/ncu_$k.log 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:f16p_gemm_pair --launch-skip 40 -c 1 -o gpurun_out/ncu_f16p_pair_tau21 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pair.log 2>&1
python tools/timeline.py --steps 1,25,50 > gpurun_out/timeline.txt 2>&1
out=gpurun_out/sweep.jsonl; : > $out
for N in 64 256 1024 4096 16384; do
  timeout 600 python bench.py --config C5 --members $N --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/sweep_err.log | tail -1 >> $out
done
for C in C1 C2; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline 2>>gpurun_out/sweep_err.log | tail -1 >> $out
done
timeout 900 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_c4.log 2>&1
