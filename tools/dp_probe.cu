// Single-SM latency probe (not part of the library): the constants that bound the shared-memory
// tail of the W-cycle -- dependent DADD / DMUL / DFMA / division chains, LDS.64, shuffles and
// bar.sync at several thread counts -- measured with clock64() on one CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/bin/dp_probe tools/dp_probe.cu && tools/bin/dp_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R = 4096;

__global__ void k_chain(double* out, long long* cyc, double a, double b, int mode) {
    double x = a + threadIdx.x;
    __syncthreads();
    long long t0 = clock64();
    switch (mode) {
        case 0:
            for (int i = 0; i < R; ++i) x = __dadd_rn(x, b);
            break;
        case 1:
            for (int i = 0; i < R; ++i) x = __dmul_rn(x, b);
            break;
        case 2:
            for (int i = 0; i < R; ++i) x = __fma_rn(x, b, a);
            break;
        case 3:
            for (int i = 0; i < R / 16; ++i) x = __ddiv_rn(x, b);
            break;
        case 4: {  // quotient from a precomputed reciprocal + two Markstein corrections
            const double y = 1.0 / b;
            for (int i = 0; i < R / 16; ++i) {
                double q = __dmul_rn(x, y);
                double r = __fma_rn(-b, q, x);
                q = __fma_rn(r, y, q);
                r = __fma_rn(-b, q, x);
                x = __fma_rn(r, y, q);
            }
            break;
        }
        case 5:
            for (int i = 0; i < R; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 0.0;
            break;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_lds(double* out, long long* cyc) {
    __shared__ long long idx[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i * 37 + 11) & 1023;
    __syncthreads();
    long long j = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) j = idx[j];
    long long t1 = clock64();
    out[threadIdx.x] = (double)j;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_bar(long long* cyc, int n) {
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
        if (n == 0)
            __syncthreads();
        else
            asm volatile("bar.sync 1, %0;" ::"r"(n) : "memory");
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// DP throughput: 8 independent chains per thread
__global__ void k_tput(double* out, long long* cyc, double b) {
    double x[8];
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x + k;
    __syncthreads();
    long long t0 = clock64();
    for (int i = 0; i < R / 8; ++i)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = __dadd_rn(x[k], b);
    __syncthreads();
    long long t1 = clock64();
    double s = 0;
    for (int k = 0; k < 8; ++k) s += x[k];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1024 * sizeof(double));
    cudaMallocManaged(&cyc, sizeof(long long));
    const char* names[] = {"DADD", "DMUL", "DFMA", "__ddiv_rn", "rcp+2 Markstein div", "SHFL(+DADD)"};
    const int per[] = {R, R, R, R / 16, R / 16, R};
    for (int m = 0; m < 6; ++m) {
        k_chain<<<1, 32>>>(out, cyc, 1.0000001, 0.99999, m);
        cudaDeviceSynchronize();
        k_chain<<<1, 32>>>(out, cyc, 1.0000001, 0.99999, m);
        cudaDeviceSynchronize();
        printf("%-22s dependent latency %.1f cycles\n", names[m], (double)*cyc / per[m]);
    }
    k_lds<<<1, 32>>>(out, cyc);
    cudaDeviceSynchronize();
    k_lds<<<1, 32>>>(out, cyc);
    cudaDeviceSynchronize();
    printf("%-22s dependent latency %.1f cycles\n", "LDS.64", (double)*cyc / R);
    for (int t : {32, 64, 256, 512, 1024}) {
        for (int named = 0; named < 2; ++named) {
            k_bar<<<1, t>>>(cyc, named ? t : 0);
            cudaDeviceSynchronize();
            k_bar<<<1, t>>>(cyc, named ? t : 0);
            cudaDeviceSynchronize();
            printf("bar.sync %s %4d threads: %.1f cycles\n", named ? "named" : "__sync", t, (double)*cyc / R);
        }
    }
    for (int t : {32, 128, 256, 512, 1024}) {
        k_tput<<<1, t>>>(out, cyc, 0.5);
        cudaDeviceSynchronize();
        k_tput<<<1, t>>>(out, cyc, 0.5);
        cudaDeviceSynchronize();
        printf("DADD throughput %4d threads: %.2f warp-instr/cycle/SM\n", t, (t / 32.0) * R / (double)*cyc);
    }
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("SM clock attribute %.0f MHz\n", clk / 1000.0);
    return 0;
}
