# Round-2 profile refresh (GPU box, repo root).  Outputs under gpurun_out/, summaries copied into
# profiles/r02/ by hand.  Each ncu command runs only after the same program exited 0 without ncu.
set -x
O=gpurun_out
B1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
# 1. noise placement A/B on the current code, interleaved (graph replay, default config C3)
for r in 1 2; do
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ab_noise_conc_$r.log 2>&1
  ENKS_NOISE_CONCURRENT=0 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/ab_noise_serial_$r.log 2>&1
done
# 2. measured per-rank kernels + modelled collectives (members sharded over 1/2/4/8 ranks)
python tools/shard_model.py --config C3 --graph > $O/shard_model_c3.log 2>&1
# 3. launch list of one C3 horizon (cold, serialised)
$B1 > $O/b1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3_h50.csv $B1 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c3_h50.csv 1 > $O/launches_c3_h50_summary.txt
# 4. ncu --set full of the kernels without an r01 summary (H=8 horizon, after warm-up launches)
B8="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --horizon 8"
for k in spd_inverse tc_gemm_kernel member_partial uchain center_f16pair_t f16p_gemm_pair; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 6 -c 1 \
    -o $O/ncu_r02_$k $B8 > $O/ncu_r02_$k.log 2>&1
  python tools/ncu_summary.py $O/ncu_r02_$k.ncu-rep > $O/ncu_r02_${k}_summary.txt 2>&1
done
# (compute-sanitizer is closed on this GPU pool: runs under it left GPUs needing a reset)
