# TMEM accumulation-chain length sweep (ENKS_TC_CHAIN) at C3, then GPU parity at the candidates.
B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
o=gpurun_out/ab_chain.txt; : > $o
for c in 8 4 16 32 64 8; do
  echo "chain=$c $(ENKS_TC_CHAIN=$c timeout 300 $B 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());k=d["kernels"];print(round(d["value"],4), round(k["cross"]["ms_per_horizon"],1), round(k["correction"]["ms_per_horizon"],2), round(k["shift"]["ms_per_horizon"],2))')" >> $o
done
for c in 16 32; do
  echo "pytest chain=$c: $(ENKS_TC_CHAIN=$c timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -1)" >> $o
done
