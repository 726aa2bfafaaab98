# Launch list and member-sum capture of the final round-2 code (GPU box, repo root).
set -x
O=gpurun_out
B1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
$B1 > $O/b1.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_c3_h50_r02i.csv $B1 > /dev/null 2>&1
python tools/launch_summary.py $O/launches_c3_h50_r02i.csv 3 > $O/launches_c3_h50_r02i_summary.txt
B8="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --horizon 8"
$B8 > $O/b8.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on \
  -k regex:member_partial2 --launch-skip 4 -c 1 -o $O/ncu_r02i_member_partial2 $B8 > $O/ncu_r02i_mp2.log 2>&1
python tools/ncu_summary.py $O/ncu_r02i_member_partial2.ncu-rep > $O/ncu_r02i_member_partial2_summary.txt 2>&1
