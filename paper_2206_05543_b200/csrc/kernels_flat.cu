// K2 for the small and middle levels: flat (non-marching) fused residual + full-weighting
// restriction, rc = restrict(b - A x) (reference multigrid.py:176-177, :104-119).
//
// The marching kernels amortise a pipeline fill over a long column of rows/planes; on levels
// of a few thousand to a million unknowns there are too few CTAs for that to pay, and each
// launch is latency-bound.  Here one CTA owns a small coarse tile, forms r on the
// (2C+1)-point fine footprint of the tile in shared memory straight from L2-resident x and b,
// and full-weights it, all in one short pass: the whole level is one wave of short CTAs.
// The expression trees are those of k_restrict / residual2d / residual3d (Appendix A.3).
#include <cstdlib>

#include "kernels.h"
#include "march.cuh"

namespace spaimg {

constexpr int F2_CH = 8, F2_CW = 32;              // 2D coarse tile (rows x cols)
constexpr int F3_CZ = 2, F3_CY = 4, F3_CX = 32;   // 3D coarse tile

template <class T>
__global__ void __launch_bounds__(256) k_rr2d_flat(Layout Lf, Layout Lc, const T* __restrict__ x,
                                                   const T* __restrict__ b, T* __restrict__ bc, T sA) {
    constexpr int RH = 2 * F2_CH + 1, RW = 2 * F2_CW + 1, RP = RW + 1;
    __shared__ T rs[RH * RP];
    const int n = Lf.n, m = Lc.n;
    const int I0 = blockIdx.y * F2_CH, J0 = blockIdx.x * F2_CW;
    const int f0 = 2 * I0, g0 = 2 * J0;  // fine interior index of local (0, 0)
    flat_stage_r<T, 2, false, RH * RW, 256, 3>(
        x, b, Lf, sA,
        [&](int q, long long& p) {
            const int i0 = f0 + q / RW, i1 = g0 + q % RW;
            p = Lf.origin + (long long)i0 * Lf.px + i1;
            return (i0 < n) & (i1 < n);
        },
        [&](int q, T rv) { rs[(q / RW) * RP + q % RW] = rv; });
    __syncthreads();
    const int yc = threadIdx.x / F2_CW, xc = threadIdx.x % F2_CW;
    const int I = I0 + yc, K = J0 + xc;
    if (I >= m || K >= m) return;
    T t[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const int c = 2 * xc + a;
        t[a] = fw<T>(rs[(2 * yc) * RP + c], rs[(2 * yc + 1) * RP + c], rs[(2 * yc + 2) * RP + c]);
    }
    bc[Lc.origin + (long long)I * Lc.px + K] = fw<T>(t[0], t[1], t[2]);
}

template <class T>
__global__ void __launch_bounds__(256) k_rr3d_flat(Layout Lf, Layout Lc, const T* __restrict__ x,
                                                   const T* __restrict__ b, T* __restrict__ bc, T sA) {
    constexpr int RZ = 2 * F3_CZ + 1, RY = 2 * F3_CY + 1, RX = 2 * F3_CX + 1, RP = RX + 1;
    __shared__ T rs[RZ * RY * RP];
    const int n = Lf.n, m = Lc.n;
    const int I0 = blockIdx.z * F3_CZ, J0 = blockIdx.y * F3_CY, K0 = blockIdx.x * F3_CX;
    const int f0 = 2 * I0, f1 = 2 * J0, f2 = 2 * K0;
    flat_stage_r<T, 3, false, RZ * RY * RX, 256, 3>(
        x, b, Lf, sA,
        [&](int q, long long& p) {
            const int lz = q / (RY * RX), rem = q - lz * RY * RX, ly = rem / RX, lx = rem - ly * RX;
            const int i0 = f0 + lz, i1 = f1 + ly, i2 = f2 + lx;
            p = Lf.origin + (long long)i0 * Lf.pp + (long long)i1 * Lf.px + i2;
            return (i0 < n) & (i1 < n) & (i2 < n);
        },
        [&](int q, T rv) {
            const int lz = q / (RY * RX), rem = q - lz * RY * RX, ly = rem / RX, lx = rem - ly * RX;
            rs[(lz * RY + ly) * RP + lx] = rv;
        });
    __syncthreads();
    const int zc = threadIdx.x / (F3_CY * F3_CX), yc = (threadIdx.x / F3_CX) % F3_CY, xc = threadIdx.x % F3_CX;
    const int I = I0 + zc, J = J0 + yc, K = K0 + xc;
    if (I >= m || J >= m || K >= m) return;
    T u[3];
#pragma unroll
    for (int qk = 0; qk < 3; ++qk) {
        T t[3];
#pragma unroll
        for (int qj = 0; qj < 3; ++qj) {
            const int o = (2 * yc + qj) * RP + 2 * xc + qk;
            t[qj] = fw<T>(rs[(2 * zc) * RY * RP + o], rs[(2 * zc + 1) * RY * RP + o], rs[(2 * zc + 2) * RY * RP + o]);
        }
        u[qk] = fw<T>(t[0], t[1], t[2]);
    }
    bc[Lc.origin + (long long)I * Lc.pp + (long long)J * Lc.px + K] = fw<T>(u[0], u[1], u[2]);
}

// ------------------------------------------------------------------------------------------
// K2 + the coarse level's first pre-sweep from zero, for the small levels: the coarse right-
// hand side bc = restrict(b - A x) is formed on the coarse tile plus a one-point ring (the
// ring recomputed from the fine footprint), and the coarse level's zero-start sweep
// xc' = 0 + omega ((M bc) sM) (r = b - A 0 = b exactly, multigrid.py:99-100) is applied to the
// tile in the same pass.  One launch per level on the way down instead of two.
// ------------------------------------------------------------------------------------------
template <class T, int S>
__global__ void __launch_bounds__(256) k_rr2d_flat_fz(Layout Lf, Layout Lc, const T* __restrict__ x,
                                                      const T* __restrict__ b, T* __restrict__ bc,
                                                      T* __restrict__ xc, Terms<T> M, T sA, T sMc, T omega) {
    using O = Op<T>;
    constexpr int BH = F2_CH + 2, BW = F2_CW + 2;          // coarse tile + ring
    constexpr int RH = 2 * BH + 1, RW = 2 * BW + 1, RP = RW + 1;  // fine r footprint
    __shared__ T rs[RH * RP];
    __shared__ T bs[BH * BW];
    const int n = Lf.n, m = Lc.n;
    const int I0 = blockIdx.y * F2_CH - 1, J0 = blockIdx.x * F2_CW - 1;  // ring origin (coarse)
    const int f0 = 2 * I0, g0 = 2 * J0;
    flat_stage_r<T, 2, false, RH * RW, 256, 3>(
        x, b, Lf, sA,
        [&](int q, long long& p) {
            const int i0 = f0 + q / RW, i1 = g0 + q % RW;
            p = Lf.origin + (long long)i0 * Lf.px + i1;
            return (i0 >= 0) & (i0 < n) & (i1 >= 0) & (i1 < n);
        },
        [&](int q, T rv) { rs[(q / RW) * RP + q % RW] = rv; });
    __syncthreads();
    for (int q = threadIdx.x; q < BH * BW; q += blockDim.x) {
        const int yc = q / BW, xc_ = q - yc * BW;
        const int I = I0 + yc, K = J0 + xc_;
        T v = T(0);  // r = b on the coarse interior, 0 outside (zero start)
        if (I >= 0 && I < m && K >= 0 && K < m) {
            T t[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int c = 2 * xc_ + a;
                t[a] = fw<T>(rs[(2 * yc) * RP + c], rs[(2 * yc + 1) * RP + c], rs[(2 * yc + 2) * RP + c]);
            }
            v = fw<T>(t[0], t[1], t[2]);
        }
        bs[q] = v;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < F2_CH * F2_CW; q += blockDim.x) {
        const int yc = q / F2_CW + 1, xc_ = q % F2_CW + 1;
        const int I = I0 + yc, K = J0 + xc_;
        if (I >= m || K >= m) continue;
        T acc = T(0);
        const int nt = tnt<T, S>(M);
#pragma unroll
        for (int k = 0; k < (S == SHAPE_GENERIC ? kMaxTerms : ShapeT<(S == SHAPE_GENERIC ? 1 : S)>::nt); ++k) {
            if (S == SHAPE_GENERIC && k >= nt) break;
            acc = O::add(acc, O::mul(M.c[k], bs[(yc + toff<T, S>(M, k, 0)) * BW + xc_ + toff<T, S>(M, k, 1)]));
        }
        const long long pc = Lc.origin + (long long)I * Lc.px + K;
        bc[pc] = bs[yc * BW + xc_];
        xc[pc] = relax<T>(T(0), acc, sMc, omega);
    }
}

template <class T, int S>
static cudaError_t rr_fz(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T* xc,
                         const Terms<T>& M, T sA, T sMc, T omega, cudaStream_t s) {
    const int m = Lc.n;
    if (Lf.dim == 2) {
        dim3 g((m + F2_CW - 1) / F2_CW, (m + F2_CH - 1) / F2_CH);
        return launch_k(k_rr2d_flat_fz<T, S>, g, dim3(256), 0, s, Lf, Lc, x, b, bc, xc, M, sA, sMc, omega);
    }
    // 3D: measured slower than two kernels (the ring recomputation costs more than the launch it
    // saves, c3 +7 %); the solver never asks for it
    return cudaErrorNotSupported;
}

template <class T>
cudaError_t launch_residual_restrict_fz(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T* xc,
                                        const Terms<T>& M, int shape, T sA, T sMc, T omega, cudaStream_t s) {
    switch (shape) {
        case SHAPE_C1: return rr_fz<T, SHAPE_C1>(Lf, Lc, x, b, bc, xc, M, sA, sMc, omega, s);
        case SHAPE_STAR5:
            if (Lf.dim == 2) return rr_fz<T, SHAPE_STAR5>(Lf, Lc, x, b, bc, xc, M, sA, sMc, omega, s);
            break;
        case SHAPE_BOX9:
            if (Lf.dim == 2) return rr_fz<T, SHAPE_BOX9>(Lf, Lc, x, b, bc, xc, M, sA, sMc, omega, s);
            break;
        case SHAPE_STAR7:
            if (Lf.dim == 3) return rr_fz<T, SHAPE_STAR7>(Lf, Lc, x, b, bc, xc, M, sA, sMc, omega, s);
            break;
        default: break;
    }
    return rr_fz<T, SHAPE_GENERIC>(Lf, Lc, x, b, bc, xc, M, sA, sMc, omega, s);
}

template cudaError_t launch_residual_restrict_fz<double>(const Layout&, const Layout&, const double*, const double*,
                                                         double*, double*, const Terms<double>&, int, double, double,
                                                         double, cudaStream_t);
template cudaError_t launch_residual_restrict_fz<float>(const Layout&, const Layout&, const float*, const float*,
                                                        float*, float*, const Terms<float>&, int, float, float, float,
                                                        cudaStream_t);

int flat_threshold(int dim) {
    const char* e = getenv(dim == 2 ? "SPAIMG_FLAT_N2" : "SPAIMG_FLAT_N3");
    if (e) return atoi(e);
    return dim == 2 ? 1024 : 64;  // measured optimum (tools/tune.py c1-c4)
}

template <class T>
cudaError_t launch_residual_restrict_flat(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T sA,
                                          cudaStream_t s) {
    const int m = Lc.n;
    if (Lf.dim == 2) {
        dim3 g((m + F2_CW - 1) / F2_CW, (m + F2_CH - 1) / F2_CH);
        return launch_k(k_rr2d_flat<T>, g, dim3(256), 0, s, Lf, Lc, x, b, bc, sA);
    } else {
        dim3 g((m + F3_CX - 1) / F3_CX, (m + F3_CY - 1) / F3_CY, (m + F3_CZ - 1) / F3_CZ);
        return launch_k(k_rr3d_flat<T>, g, dim3(256), 0, s, Lf, Lc, x, b, bc, sA);
    }
    return cudaGetLastError();
}

template cudaError_t launch_residual_restrict_flat<double>(const Layout&, const Layout&, const double*, const double*,
                                                           double*, double, cudaStream_t);
template cudaError_t launch_residual_restrict_flat<float>(const Layout&, const Layout&, const float*, const float*,
                                                          float*, float, cudaStream_t);

}  // namespace spaimg
