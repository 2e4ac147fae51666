// Cluster-barrier latency probe: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/clprobe tools/cluster_probe.cu
#include <cstdio>
#include <cooperative_groups.h>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void k_cl(int n, double* buf) {
    cg::cluster_group cl = cg::this_cluster();
    double v = 0;
    for (int i = 0; i < n; ++i) {
        // touch global memory written by another CTA of the cluster
        const int r = cl.block_rank();
        if (threadIdx.x == 0) buf[r] = v + i;
        cl.sync();
        v += __ldcg(&buf[(r + 1) % cl.num_blocks()]);
    }
    if (v < -1) buf[0] = v;
}
int main() {
    double* buf; cudaMalloc(&buf, 4096);
    cudaStream_t s; cudaStreamCreate(&s);
    for (int cs : {2, 8, 16}) {
        for (int thr : {256, 1024}) {
            cudaLaunchConfig_t cfg{}; cfg.gridDim = dim3(cs); cfg.blockDim = dim3(thr); cfg.stream = s;
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            if (cs > 8) cudaFuncSetAttribute(k_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            int n = 2000;
            cudaError_t e = cudaLaunchKernelEx(&cfg, k_cl, 10, buf); cudaStreamSynchronize(s);
            if (e != cudaSuccess) { printf("cluster %d: %s\n", cs, cudaGetErrorString(e)); continue; }
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a, s); cudaLaunchKernelEx(&cfg, k_cl, n, buf); cudaEventRecord(b, s); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("cluster %2d x %4d threads: %.3f us per cluster.sync (+ L2 round trip)\n", cs, thr, ms * 1e3 / n);
        }
    }
}
