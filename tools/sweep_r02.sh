# Round-2 sweep (GPU box, repo root): interleaved chain-length A/B of the f16p contraction, the
# paper's Table-1 shapes, C5 ensemble sweep, C1/C2 lines, C4 on one B200.
set -x
O=gpurun_out
Q="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e"
: > $O/ab_chain_r02.jsonl
for r in 1 2 3; do
  for c in 16 8; do
    ENKS_F16P_CHAIN=$c python bench.py $Q 2>/dev/null | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(json.dumps({'chain': $c, 'run': $r, 'value': d['value'], 'cross_ms': d['kernels']['cross']['ms_per_horizon'], 'sm_mhz': d['clocks']['sm_mhz']}))" >> $O/ab_chain_r02.jsonl
  done
done
python tools/table1.py > $O/table1.log 2>&1
out=$O/sweep_r02.jsonl; : > $out
for N in 64 256 1024 4096 16384; do
  timeout 900 python bench.py --config C5 --members $N --steps 3 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
for C in C1 C2; do
  timeout 600 python bench.py --config $C --steps 5 --warmup 3 --no-cpu-baseline 2>>$O/sweep_err.log | tail -1 >> $out
done
timeout 1200 python bench.py --config C4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_c4.log 2>&1
