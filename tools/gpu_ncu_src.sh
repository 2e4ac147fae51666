# one eager-run ncu --set full capture with source: bash tools/gpu_ncu_src.sh <name> <demangled kernel regex> <skip> <prof_op args...>
# writes gpurun_out/<name>.{raw,source}.csv and prints the headline metrics + the hottest source lines
mkdir -p gpurun_out
name=$1; rx=$2; skip=$3; shift 3
SPAIMG_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -f --kernel-name-base demangled \
  -k "regex:$rx" -s $skip -c 1 -o gpurun_out/$name python tools/prof_op.py "$@" > gpurun_out/$name.log 2>&1; echo ncu_$name=$?
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$name.source.csv 2>/dev/null
rm -f gpurun_out/$name.ncu-rep
python - <<PY
import csv
rows = list(csv.reader(open("gpurun_out/$name.raw.csv")))
h, u, v = rows[0], rows[1], rows[2]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__bytes.sum.per_second",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers"]
for w in want:
    if w in h:
        i = h.index(w)
        print(f"{w}: {v[i][:90]} {u[i]}")
PY
python tools/src_hot.py gpurun_out/$name.source.csv 28
