# compute-sanitizer tier: every kernel family on small grids (tools/sanitize_case.py) under each
# tool, with the marching kernels forced on every level (FLAT=0) and with the default flat kernels.
#   bash tools/gpu_sanitize.sh  -> gpurun_out/sanitize_<tool>_<mode>.log
mkdir -p gpurun_out
for mode in march flat; do
  if [ $mode = march ]; then export SPAIMG_FLAT_N2=0 SPAIMG_FLAT_N3=0; else unset SPAIMG_FLAT_N2 SPAIMG_FLAT_N3; fi
  for tool in memcheck racecheck synccheck initcheck; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report all"
    timeout 1800 compute-sanitizer --tool $tool $extra --error-exitcode 17 --print-limit 50 \
      python tools/sanitize_case.py > gpurun_out/sanitize_${tool}_${mode}.log 2>&1
    echo "$tool $mode rc=$?"
  done
done
