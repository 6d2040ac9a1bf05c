# ncu launch lists (dram bytes + time per launch) of one host-loop hull per config
for cfg in "unit-square 1000000 C1" "on-circle 10000000 C3" "near-circle 10000000 C3n" "unit-cube 10000000 C4c" "uniform-ball 10000000 C4b"; do
  set -- $cfg
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/tr_$3.csv python tools/ncu_round.py $1 $2 > /dev/null 2>&1
done
