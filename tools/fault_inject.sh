# Self-test of the checked build (sanitizer-substitute tier): link a library whose compile-time
# coarse engine lacks the barrier before the prolongation (-DSPAIMG_DEBUG_BREAK_BARRIER) and run
# the sanitizer workload against it; every run must FAIL (bitwise mismatch with the C oracle).
#   bash tools/fault_inject.sh            (build here, then on the GPU box:)
#   for i in 1 2 3; do SPAIMG_LIB_OVERRIDE=$PWD/tools/bin/broken/lib_jit.so python tools/sanitize_case.py; done
set -e
python -m paper_2206_05543_b200.build --debug > /dev/null
mkdir -p tools/bin/broken /tmp/spaimg_broken
cp paper_2206_05543_b200/build/debug/*.o /tmp/spaimg_broken/
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --fmad=false -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden -DSPAIMG_DEBUG_CHECKS -DSPAIMG_DEBUG_BREAK_BARRIER -I include \
  -I paper_2206_05543_b200/csrc -c paper_2206_05543_b200/csrc/kernels_tail_fast2d.cu \
  -o /tmp/spaimg_broken/kernels_tail_fast2d.o
nvcc -gencode arch=compute_100a,code=sm_100a -shared -Xcompiler -fPIC -o tools/bin/broken/lib_jit.so /tmp/spaimg_broken/*.o
echo tools/bin/broken/lib_jit.so
