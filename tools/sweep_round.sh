# C5 ensemble-size sweep + C1/C2 lines + ncu capture of the CTA-pair cross-moment kernel
out=gpurun_out/sweep.jsonl; : > $out
for N in 64 256 1024 4096 16384; do
  timeout 600 python bench.py --config C5 --members $N --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>gpurun_out/sweep_err.log | tail -1 >> $out
done
for C in C1 C2; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline 2>>gpurun_out/sweep_err.log | tail -1 >> $out
done
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log >> $out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:f16p_gemm_pair --launch-skip 40 -c 1 -o gpurun_out/ncu_f16p_pair python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_pair.log 2>&1
tail -2 gpurun_out/ncu_pair.log
