mkdir -p gpurun_out
for v in nojit; do for i in 1 2 3 4 5; do
  SPAIMG_LIB_OVERRIDE=$PWD/tools/bin/broken/lib_$v.so timeout 600 python tools/sanitize_case.py > gpurun_out/broken_${v}_$i.log 2>&1; echo "$v $i rc=$?"
done; done
