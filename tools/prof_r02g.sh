# Round-2 final check after the noise replay and the staged shift epilogue (GPU box, repo root).
# Outputs under gpurun_out/, summaries copied into profiles/r02/ by hand.  Each ncu command runs
# only after the same program exited 0 without ncu.
set -x
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu_r02g.log 2>&1; tail -2 $O/pytest_gpu_r02g.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02g.log 2>&1; tail -2 $O/smoke_r02g.log
for r in 1 2; do python bench.py > $O/bench_c3_r02g_$r.json 2> $O/bench_c3_r02g_$r.err; done
out=$O/sweep_r02g.jsonl; : > $out
for N in 64 128 256 1024; do
  timeout 900 python bench.py --config C5 --members $N --steps 3 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
python tools/shard_model.py --config C3 --graph > $O/shard_model_c3_r02g.log 2>&1
B8="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --horizon 8"
$B8 > $O/b8.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
  --kernel-name-base mangled -k regex:pair_kernelILb1 --launch-skip 2 -c 1 \
  -o $O/ncu_r02g_shift $B8 > $O/ncu_r02g_shift.log 2>&1
python tools/ncu_summary.py $O/ncu_r02g_shift.ncu-rep > $O/ncu_r02g_shift_summary.txt 2>&1
