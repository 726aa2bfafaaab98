# Round-2 final validation after the one-pass member sums (GPU box, repo root).
set -x
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > $O/pytest_gpu_r02h.log 2>&1; tail -2 $O/pytest_gpu_r02h.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke_r02h.log 2>&1; tail -2 $O/smoke_r02h.log
for r in 1 2; do python bench.py > $O/bench_c3_r02h_$r.json 2> $O/bench_c3_r02h_$r.err; done
out=$O/sweep_r02h.jsonl; : > $out
for N in 64 128 256 1024; do
  timeout 900 python bench.py --config C5 --members $N --steps 3 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
python tools/shard_model.py --config C3 --graph > $O/shard_model_c3_r02h.log 2>&1
