# usage: bash tools/gpu_prof.sh <tag> <kind> <n> [kregex] [skip] [count]
TAG=$1; KIND=$2; N=$3; KRE=${4:-k_round}; SKIP=${5:-13}; CNT=${6:-3}
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python tools/prof_run.py --kind $KIND --n $N --reps 2 --hostloop 1 > gpurun_out/prof_run_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c $CNT -o gpurun_out/prof_$TAG python tools/prof_run.py --kind $KIND --n $N --reps 2 --hostloop 1 > gpurun_out/ncu_full_$TAG.log 2>&1
