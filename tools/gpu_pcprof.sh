mkdir -p gpurun_out
SPAIMG_NO_GRAPH=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -s 60 -c 40 --csv --log-file gpurun_out/warm_c2_pc.csv python tools/prof_op.py c2 9 4 > /dev/null 2>&1; echo warm=$?
timeout 600 ncu --set full --clock-control none --import-source on -f -k regex:"k_sweep2d_march<double, 3, 0, 3>" -s 3 -c 1 -o gpurun_out/full_pc python tools/prof_op.py c2 9 2 > gpurun_out/ncu_pc.log 2>&1; echo full=$?
