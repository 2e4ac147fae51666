// K1 fused smoothing sweep and K2 fused residual + restriction.
//
// Sweep (reference multigrid.py:98-100 for one step):  r = b - A x on the tile plus a one-point
// halo in shared memory, then x' = x + omega * ((M r) * sM) from that tile in the same pass.
// r is forced to zero outside the interior (the reference zero-pads r itself, stencils.py:146).
#include "sweep2d_march.cuh"

namespace spaimg {

__device__ __forceinline__ long long pidx2(const Layout& L, int i0, int i1) { return L.origin + (long long)i0 * L.px + i1; }
__device__ __forceinline__ long long pidx3(const Layout& L, int i0, int i1, int i2) {
    return L.origin + (long long)i0 * L.pp + (long long)i1 * L.px + i2;
}

// ------------------------------------------------------------------------------------------
// v1 tiles (halo recomputation; row/plane marching versions replace these per dim)
// ------------------------------------------------------------------------------------------
constexpr int S2_TW = 64, S2_TH = 16;
constexpr int S3_TX = 32, S3_TY = 8, S3_TZ = 4;

// NORM: ||b - A x||^2 of the INPUT iterate over the tile's own points joins the deterministic
// norm reduction (march.cuh norm_epilogue): part A of the solve loop on flat-sized finest levels
template <class T, int S, bool FZ, bool NORM = false>
__global__ void __launch_bounds__(256) k_sweep2d_tile(Layout L, const T* __restrict__ x, const T* __restrict__ b,
                                                      T* __restrict__ xo, Terms<T> M, T sA, T sM, T omega,
                                                      NormOut no) {
    using O = Op<T>;
    constexpr int RW = S2_TW + 2, RH = S2_TH + 2;
    __shared__ T rs[RH * RW];
    const int c0 = blockIdx.x * S2_TW, r0 = blockIdx.y * S2_TH;
    const int n = L.n;
    double nacc = 0.0;
    flat_stage_r<T, 2, FZ, RH * RW, 256, 3>(
        x, b, L, sA,
        [&](int q, long long& p) {
            const int i0 = r0 - 1 + q / RW, i1 = c0 - 1 + q % RW;
            p = pidx2(L, i0, i1);
            return (i0 >= 0) & (i0 < n) & (i1 >= 0) & (i1 < n);
        },
        [&](int q, T rv) {
            rs[q] = rv;
            if constexpr (NORM) {
                const int lr = q / RW, lc = q % RW;  // the one-point ring belongs to the neighbour tiles
                if (lr >= 1 && lr <= S2_TH && lc >= 1 && lc <= S2_TW) nacc += (double)rv * (double)rv;
            }
        });
    __syncthreads();
    for (int q = threadIdx.x; q < S2_TH * S2_TW; q += blockDim.x) {
        const int a0 = q / S2_TW, a1 = q % S2_TW;
        const int i0 = r0 + a0, i1 = c0 + a1;
        if (i0 >= n || i1 >= n) continue;
        T acc = T(0);
        const int nt = tnt<T, S>(M);
#pragma unroll
        for (int k = 0; k < (S == SHAPE_GENERIC ? kMaxTerms : ShapeT<(S == SHAPE_GENERIC ? 1 : S)>::nt); ++k) {
            if (S == SHAPE_GENERIC && k >= nt) break;
            const int o0 = toff<T, S>(M, k, 0), o1 = toff<T, S>(M, k, 1);
            acc = O::add(acc, O::mul(M.c[k], rs[(a0 + 1 + o0) * RW + (a1 + 1 + o1)]));
        }
        const long long p = pidx2(L, i0, i1);
        xo[p] = relax<T>(FZ ? T(0) : x[p], acc, sM, omega);
    }
    if constexpr (NORM) norm_epilogue(nacc, no);
}

template <class T, int S, bool FZ, bool NORM = false>
__global__ void __launch_bounds__(256) k_sweep3d_tile(Layout L, const T* __restrict__ x, const T* __restrict__ b,
                                                      T* __restrict__ xo, Terms<T> M, T sA, T sM, T omega,
                                                      NormOut no) {
    using O = Op<T>;
    constexpr int RX = S3_TX + 2, RY = S3_TY + 2, RZ = S3_TZ + 2;
    __shared__ T rs[RZ * RY * RX];
    const int x0 = blockIdx.x * S3_TX, y0 = blockIdx.y * S3_TY, z0 = blockIdx.z * S3_TZ;
    const int n = L.n;
    double nacc = 0.0;
    flat_stage_r<T, 3, FZ, RZ * RY * RX, 256, 3>(
        x, b, L, sA,
        [&](int q, long long& p) {
            const int i0 = z0 - 1 + q / (RY * RX), i1 = y0 - 1 + (q / RX) % RY, i2 = x0 - 1 + q % RX;
            p = pidx3(L, i0, i1, i2);
            return (i0 >= 0) & (i0 < n) & (i1 >= 0) & (i1 < n) & (i2 >= 0) & (i2 < n);
        },
        [&](int q, T rv) {
            rs[q] = rv;
            if constexpr (NORM) {
                const int lz = q / (RY * RX), ly = (q / RX) % RY, lx = q % RX;
                if (lz >= 1 && lz <= S3_TZ && ly >= 1 && ly <= S3_TY && lx >= 1 && lx <= S3_TX)
                    nacc += (double)rv * (double)rv;
            }
        });
    __syncthreads();
    for (int q = threadIdx.x; q < S3_TZ * S3_TY * S3_TX; q += blockDim.x) {
        const int a0 = q / (S3_TY * S3_TX), a1 = (q / S3_TX) % S3_TY, a2 = q % S3_TX;
        const int i0 = z0 + a0, i1 = y0 + a1, i2 = x0 + a2;
        if (i0 >= n || i1 >= n || i2 >= n) continue;
        T acc = T(0);
        const int nt = tnt<T, S>(M);
#pragma unroll
        for (int k = 0; k < (S == SHAPE_GENERIC ? kMaxTerms : ShapeT<(S == SHAPE_GENERIC ? 1 : S)>::nt); ++k) {
            if (S == SHAPE_GENERIC && k >= nt) break;
            const int o0 = toff<T, S>(M, k, 0), o1 = toff<T, S>(M, k, 1), o2 = toff<T, S>(M, k, 2);
            acc = O::add(acc, O::mul(M.c[k], rs[((a0 + 1 + o0) * RY + (a1 + 1 + o1)) * RX + (a2 + 1 + o2)]));
        }
        const long long p = pidx3(L, i0, i1, i2);
        xo[p] = relax<T>(FZ ? T(0) : x[p], acc, sM, omega);
    }
    if constexpr (NORM) norm_epilogue(nacc, no);
}

bool sweep_fused_supported(int dim, int shape) {
    if (dim == 2) return shape == SHAPE_GENERIC || shape == SHAPE_C1 || shape == SHAPE_STAR5 || shape == SHAPE_BOX9;
    return shape == SHAPE_GENERIC || shape == SHAPE_C1 || shape == SHAPE_STAR7;
}

template <class T, int S, bool FZ, int NM>
cudaError_t launch_sweep3d_march(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA, T sM,
                                 T omega, const NormOut& no, cudaStream_t s, const Layout* Lc = nullptr,
                                 const T* ec = nullptr);

template <class T, int S, bool FZ, int NM>
static cudaError_t sweep_dispatch(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA, T sM,
                                  T omega, const NormOut& no, cudaStream_t s) {
    constexpr int S3 = (S == SHAPE_GENERIC || S == SHAPE_C1 || S == SHAPE_STAR7) ? S : SHAPE_GENERIC;
    // flat-sized levels: the tile kernels (with the norm when this is part A of the solve loop)
    const bool flat = (NM == 0 || NM == 1) && L.N <= flat_threshold(L.dim);
    if (L.dim == 2) {
        if (flat) {
            dim3 g((L.n + S2_TW - 1) / S2_TW, (L.n + S2_TH - 1) / S2_TH);
            return launch_k(k_sweep2d_tile<T, S, FZ, NM == 1>, g, dim3(256), 0, s, L, x, b, xo, M, sA, sM, omega, no);
        }
        return launch_sweep2d_march<T, S, FZ, NM>(L, x, b, xo, M, sA, sM, omega, no, s);
    }
    if (flat) {
        dim3 g((L.n + S3_TX - 1) / S3_TX, (L.n + S3_TY - 1) / S3_TY, (L.n + S3_TZ - 1) / S3_TZ);
        return launch_k(k_sweep3d_tile<T, S, FZ, NM == 1>, g, dim3(256), 0, s, L, x, b, xo, M, sA, sM, omega, no);
    }
    return launch_sweep3d_march<T, S3, FZ, NM>(L, x, b, xo, M, sA, sM, omega, no, s);
}

template <class T, int S>
static cudaError_t sweep_fz(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA, T sM, T omega,
                            bool fz, const NormOut* no, cudaStream_t s) {
    const NormOut n0{};
    if (no)
        return fz ? sweep_dispatch<T, S, true, 1>(L, x, b, xo, M, sA, sM, omega, *no, s)
                  : sweep_dispatch<T, S, false, 1>(L, x, b, xo, M, sA, sM, omega, *no, s);
    return fz ? sweep_dispatch<T, S, true, 0>(L, x, b, xo, M, sA, sM, omega, n0, s)
              : sweep_dispatch<T, S, false, 0>(L, x, b, xo, M, sA, sM, omega, n0, s);
}

template <class T>
cudaError_t launch_sweep(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, int shape, T sA, T sM,
                         T omega, bool from_zero, cudaStream_t s, const NormOut* no) {
    switch (shape) {
        case SHAPE_C1: return sweep_fz<T, SHAPE_C1>(L, x, b, xo, M, sA, sM, omega, from_zero, no, s);
        case SHAPE_STAR5:
            if (L.dim == 2) return sweep_fz<T, SHAPE_STAR5>(L, x, b, xo, M, sA, sM, omega, from_zero, no, s);
            break;
        case SHAPE_BOX9:
            if (L.dim == 2) return sweep_fz<T, SHAPE_BOX9>(L, x, b, xo, M, sA, sM, omega, from_zero, no, s);
            break;
        case SHAPE_STAR7:
            if (L.dim == 3) return sweep_fz<T, SHAPE_STAR7>(L, x, b, xo, M, sA, sM, omega, from_zero, no, s);
            break;
        default: break;
    }
    return sweep_fz<T, SHAPE_GENERIC>(L, x, b, xo, M, sA, sM, omega, from_zero, no, s);
}

// residual norm alone through the marching machinery (no smoothing output)
template <class T>
cudaError_t launch_norm_march(const Layout& L, const T* x, const T* b, T sA, const NormOut& no, cudaStream_t s) {
    const Terms<T> none{};
    if (L.dim == 2) return launch_sweep2d_march<T, SHAPE_C1, false, 2>(L, x, b, nullptr, none, sA, T(0), T(0), no, s);
    return launch_sweep3d_march<T, SHAPE_C1, false, 2>(L, x, b, nullptr, none, sA, T(0), T(0), no, s);
}

// ------------------------------------------------------------------------------------------
// K2 dispatch: flat tile kernels on small levels, the row march in 2D, the plane march in 3D
// ------------------------------------------------------------------------------------------
template <class T>
cudaError_t launch_residual_restrict2d_march(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T sA,
                                             cudaStream_t s);

template <class T>
cudaError_t launch_residual_restrict(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T sA,
                                     cudaStream_t s) {
    if (Lf.N <= flat_threshold(Lf.dim)) return launch_residual_restrict_flat<T>(Lf, Lc, x, b, bc, sA, s);
    if (Lf.dim == 2) return launch_residual_restrict2d_march<T>(Lf, Lc, x, b, bc, sA, s);
    const Terms<T> none{};
    return launch_sweep3d_march<T, SHAPE_C1, false, 3>(Lf, x, b, bc, none, sA, T(0), T(0), NormOut{}, s, &Lc);
}

template cudaError_t launch_sweep<double>(const Layout&, const double*, const double*, double*, const Terms<double>&,
                                          int, double, double, double, bool, cudaStream_t, const NormOut*);
template cudaError_t launch_sweep<float>(const Layout&, const float*, const float*, float*, const Terms<float>&, int,
                                         float, float, float, bool, cudaStream_t, const NormOut*);
template cudaError_t launch_norm_march<double>(const Layout&, const double*, const double*, double, const NormOut&,
                                               cudaStream_t);
template cudaError_t launch_norm_march<float>(const Layout&, const float*, const float*, float, const NormOut&,
                                              cudaStream_t);
template cudaError_t launch_residual_restrict<double>(const Layout&, const Layout&, const double*, const double*,
                                                      double*, double, cudaStream_t);
template cudaError_t launch_residual_restrict<float>(const Layout&, const Layout&, const float*, const float*, float*,
                                                     float, cudaStream_t);

}  // namespace spaimg
