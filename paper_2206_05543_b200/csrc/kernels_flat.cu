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
    pdl_wait();
    pdl_trigger();
    const int n = Lf.n, m = Lc.n;
    const int I0 = blockIdx.y * F2_CH, J0 = blockIdx.x * F2_CW;
    const int f0 = 2 * I0, g0 = 2 * J0;  // fine interior index of local (0, 0)
    for (int q = threadIdx.x; q < RH * RW; q += blockDim.x) {
        const int lr = q / RW, lc = q - lr * RW;
        const int i0 = f0 + lr, i1 = g0 + lc;
        T rv = T(0);
        if (i0 < n && i1 < n) {
            const long long p = Lf.origin + (long long)i0 * Lf.px + i1;
            rv = residual2d<T>(b[p], x[p], x[p + Lf.px], x[p - Lf.px], x[p + 1], x[p - 1], sA);
        }
        rs[lr * RP + lc] = rv;
    }
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
    pdl_wait();
    pdl_trigger();
    const int n = Lf.n, m = Lc.n;
    const int I0 = blockIdx.z * F3_CZ, J0 = blockIdx.y * F3_CY, K0 = blockIdx.x * F3_CX;
    const int f0 = 2 * I0, f1 = 2 * J0, f2 = 2 * K0;
    for (int q = threadIdx.x; q < RZ * RY * RX; q += blockDim.x) {
        const int lz = q / (RY * RX), rem = q - lz * RY * RX, ly = rem / RX, lx = rem - ly * RX;
        const int i0 = f0 + lz, i1 = f1 + ly, i2 = f2 + lx;
        T rv = T(0);
        if (i0 < n && i1 < n && i2 < n) {
            const long long p = Lf.origin + (long long)i0 * Lf.pp + (long long)i1 * Lf.px + i2;
            rv = residual3d<T>(b[p], x[p], x[p + Lf.pp], x[p - Lf.pp], x[p + Lf.px], x[p - Lf.px], x[p + 1], x[p - 1],
                               sA);
        }
        rs[(lz * RY + ly) * RP + lx] = rv;
    }
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

bool pdl_enabled() {
    static int on = -1;
    if (on < 0) {
        // measured neutral-to-slightly-negative on the c1-c4 cycles (launch latency is not the
        // bottleneck of the small levels; their memory latency is), so opt-in
        const char* e = getenv("SPAIMG_PDL");
        on = (e && e[0] == '1') ? 1 : 0;
    }
    return on == 1;
}

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
        return launch_pdl(k_rr2d_flat<T>, g, dim3(256), 0, s, Lf, Lc, x, b, bc, sA);
    } else {
        dim3 g((m + F3_CX - 1) / F3_CX, (m + F3_CY - 1) / F3_CY, (m + F3_CZ - 1) / F3_CZ);
        return launch_pdl(k_rr3d_flat<T>, g, dim3(256), 0, s, Lf, Lc, x, b, bc, sA);
    }
    return cudaGetLastError();
}

template cudaError_t launch_residual_restrict_flat<double>(const Layout&, const Layout&, const double*, const double*,
                                                           double*, double, cudaStream_t);
template cudaError_t launch_residual_restrict_flat<float>(const Layout&, const Layout&, const float*, const float*,
                                                          float*, float, cudaStream_t);

}  // namespace spaimg
