# one ncu --set full capture, exported to CSV: bash tools/gpu_ncu1.sh <name> <kernel regex> <skip> <prof_op args...>
mkdir -p gpurun_out
name=$1; rx=$2; skip=$3; shift 3
timeout 600 ncu --set full --clock-control none --import-source on -f -k "regex:$rx" -s $skip -c 1 -o gpurun_out/$name python tools/prof_op.py "$@" > gpurun_out/$name.log 2>&1; echo ncu_$name=$?
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page source --csv > gpurun_out/$name.source.csv 2>/dev/null
rm -f gpurun_out/$name.ncu-rep
