// Per-op latency probe for the shared-memory coarse engine (not part of the library): cycles of
// one "barrier + shared-memory stencil op" step on 2 warps, for
//   (a) one small op body in a loop (warm instruction cache),
//   (b) the same body chosen through a switch among NB distinct op bodies, round-robin, so every
//       step runs code that was last executed NB steps ago (instruction-cache pressure),
// plus the cost of an indexed constant-bank load (LDC) and of a dependent shared-memory load.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -Ipaper_2206_05543_b200/csrc -Iinclude \
//        -o tools/bin/op_probe tools/op_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int STEPS = 2048;

struct Params {
    int idx[4096];
};

template <int V>
__device__ __forceinline__ void body(double* s, int p, double sA) {
    // residual-like chain on one point: 5 loads, 6 dependent DP ops, 1 store (+ V to make bodies distinct)
    const double xc = s[p], xn = s[p - 64], xs = s[p + 64], xe = s[p + 1], xw = s[p - 1];
    double acc = __dadd_rn(0.0, __dmul_rn(4.0 + V, xc));
    acc = __dsub_rn(acc, xs);
    acc = __dsub_rn(acc, xn);
    acc = __dsub_rn(acc, xe);
    acc = __dsub_rn(acc, xw);
    s[p + 2048] = __dsub_rn(1.0, __dmul_rn(acc, sA));
}

template <int NB>
__device__ __forceinline__ void dispatch(int k, double* s, int p, double sA) {
    if constexpr (NB > 0) {
        if (k == NB - 1) {
            body<NB>(s, p, sA);
            return;
        }
        dispatch<NB - 1>(k, s, p, sA);
    }
}

template <int NB>
__global__ void k_ops(long long* cyc, double sA) {
    __shared__ double s[5000];
    for (int i = threadIdx.x; i < 5000; i += blockDim.x) s[i] = 1.0 / (i + 1);
    __syncthreads();
    const int p = 100 + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < STEPS; ++i) {
        asm volatile("bar.sync 1, 64;" ::: "memory");
        dispatch<NB>(i % NB, s, p, sA);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void k_ldc(long long* cyc, const __grid_constant__ Params P) {
    int j = threadIdx.x & 1;
    long long t0 = clock64();
    for (int i = 0; i < STEPS; ++i) j = P.idx[(j + i) & 4095] & 4095;  // dependent indexed LDC
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0 + (j == 12345);
}

int main_ops(long long* cyc) {
    auto run = [&](auto kern, const char* name) {
        kern<<<1, 64>>>(cyc, 0.25);
        cudaDeviceSynchronize();
        kern<<<1, 64>>>(cyc, 0.25);
        cudaDeviceSynchronize();
        printf("%-40s %.1f cycles/step\n", name, (double)*cyc / STEPS);
    };
    run(k_ops<1>, "1 body (warm)");
    run(k_ops<4>, "4 bodies round-robin");
    run(k_ops<16>, "16 bodies round-robin");
    run(k_ops<64>, "64 bodies round-robin");
    run(k_ops<160>, "160 bodies round-robin");
    Params P;
    for (int i = 0; i < 4096; ++i) P.idx[i] = (i * 97 + 13) & 4095;
    k_ldc<<<1, 64>>>(cyc, P);
    cudaDeviceSynchronize();
    k_ldc<<<1, 64>>>(cyc, P);
    cudaDeviceSynchronize();
    printf("%-40s %.1f cycles/step\n", "dependent indexed LDC (16 KB params)", (double)*cyc / STEPS);
    return 0;
}
void coarse_probe(long long* cyc);
void tailop_probe(long long* cyc);

// ---- the engine's coarse solve (tail_ops.cuh coarse_fast) in isolation, one thread ----
#include "tail_ops.cuh"
template <int NLU, bool EXACT>
__global__ void k_coarse(long long* cyc, const double* lu) {
    __shared__ double sm[2048];
    __shared__ int ci[64];
    for (int i = threadIdx.x; i < NLU * NLU + 2 * NLU; i += blockDim.x) sm[i] = lu[i];
    for (int i = threadIdx.x; i < NLU; i += blockDim.x) {
        ci[i] = 1024 + i;
        ci[NLU + i] = 1100 + i;
        sm[1024 + i] = 1.0 + 0.1 * i;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    long long t0 = clock64();
    for (int r = 0; r < 64; ++r) {
        if (EXACT)
            spaimg::coarse_exact<double, NLU>(sm, ci, sm, sm);
        else
            spaimg::coarse_fast<double, NLU>(sm, ci, sm, sm);
        __syncwarp();
    }
    long long t1 = clock64();
    cyc[0] = t1 - t0;
}

void coarse_probe(long long* cyc) {
    // a diagonally dominant LU with unit-ish pivots: -L / -U entries small, U_jj 4, 1/U_jj exact
    double h[2048];
    for (int n : {9, 27}) {
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) h[i * n + j] = i == j ? 0.0 : -0.01 * ((i + j) % 5);
        for (int j = 0; j < n; ++j) {
            h[n * n + j] = 4.0 + 0.5 * (j % 3);
            h[n * n + n + j] = 1.0 / h[n * n + j];
        }
        double* d;
        cudaMalloc(&d, sizeof(h));
        cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
        for (int rep = 0; rep < 2; ++rep) {
            if (n == 9) k_coarse<9, false><<<1, 32>>>(cyc, d); else k_coarse<27, false><<<1, 32>>>(cyc, d);
            cudaDeviceSynchronize();
        }
        printf("coarse_fast NLU=%2d                       %.1f cycles/solve\n", n, (double)*cyc / 64);
        for (int rep = 0; rep < 2; ++rep) {
            if (n == 9) k_coarse<9, true><<<1, 32>>>(cyc, d); else k_coarse<27, true><<<1, 32>>>(cyc, d);
            cudaDeviceSynchronize();
        }
        printf("coarse_exact NLU=%2d                      %.1f cycles/solve\n", n, (double)*cyc / 64);
        cudaFree(d);
    }
}

int main() {
    long long* cyc;
    cudaMallocManaged(&cyc, sizeof(long long));
    main_ops(cyc);
    coarse_probe(cyc);
    tailop_probe(cyc);
    return 0;
}

// ---- the engine's point ops (tail_ops.cuh) in a warm loop: one op + the barrier, per step ----
template <int WHICH>
__global__ void k_tailop(long long* cyc, int reps) {
    extern __shared__ double arr[];
    using namespace spaimg;
    // level n = 7 (W = 8, frame 1): x, b, r arrays of 81 elements; coarse n = 3 (x, b, 25 elements)
    TailLv<double> f{7, 3, 9, 0, 10, 91 + 10, 182 + 10, 0, 64.0, 1.0 / 64};
    TailLv<double> c{3, 2, 5, 0, 273 + 6, 298 + 6, -1, 0, 16.0, 1.0 / 16};
    for (int i = threadIdx.x; i < 400; i += blockDim.x) arr[i] = (i % 7) * 0.125;
    Terms<double> M{};
    M.nt = 9;
    for (int k = 0; k < 9; ++k) M.c[k] = 0.1 * (k + 1);
    __syncthreads();
    const int warp = threadIdx.x >> 5;
    long long t0 = clock64();
    for (int i = 0; i < reps; ++i) {
        asm volatile("bar.sync 1, 64;" ::: "memory");
        if (WHICH == 0) op_res<double, 2, 3>(f, arr);
        if (WHICH == 1) op_relax<double, SHAPE_BOX9, 2, 3, false>(f, arr, M, 0.5);
        if (WHICH == 2) op_prolong<double, 2, 3>(f, c, arr);
        if (WHICH == 3 && warp == 0) op_resfw<double, 2, 3>(f, c, arr);
        if (WHICH == 4) op_prolong_res<double, 2, 3>(f, c, arr);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

void tailop_probe(long long* cyc) {
    const char* names[] = {"RES n=7 (2 warps)", "RELAX m9 n=7", "PROLONG n=7", "RESFW n=7 (1 warp)", "PRORES n=7"};
    for (int w = 0; w < 5; ++w) {
        for (int rep = 0; rep < 2; ++rep) {
            switch (w) {
                case 0: k_tailop<0><<<1, 64, 400 * 8>>>(cyc, 256); break;
                case 1: k_tailop<1><<<1, 64, 400 * 8>>>(cyc, 256); break;
                case 2: k_tailop<2><<<1, 64, 400 * 8>>>(cyc, 256); break;
                case 3: k_tailop<3><<<1, 64, 400 * 8>>>(cyc, 256); break;
                case 4: k_tailop<4><<<1, 64, 400 * 8>>>(cyc, 256); break;
            }
            cudaDeviceSynchronize();
        }
        printf("%-40s %.1f cycles/step\n", names[w], (double)*cyc / 256);
    }
}
