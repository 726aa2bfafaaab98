B="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
o=gpurun_out/ab_noise.txt; : > $o
for cfg in "ENKS_NOISE_CONCURRENT=1" "ENKS_NOISE_CONCURRENT=0" "ENKS_NOISE_IN_CNN=1" "ENKS_NOISE_IN_CNN=3" "ENKS_NOISE_CONCURRENT=1"; do
  echo "$cfg $(env $cfg timeout 300 $B 2>&1 | tail -1 | python -c 'import json,sys;d=json.loads(sys.stdin.read());k=d["kernels"];print(round(d["value"],4), round(k["forecast"]["ms_per_horizon"],1), round(k["noise"]["ms_per_horizon"],1))')" >> $o
done
