set -x
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/b.log 2>&1; tail -1 gpurun_out/b.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_h50.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --horizon 8"
for k in noise spd_inverse center_f16pair cnn3_tc tc_gemm_kernel; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 6 -c 1 -o gpurun_out/ncu_$k $B > gpurun_out/ncu_$k.log 2>&1; tail -1 gpurun_out/ncu_$k.log
done
