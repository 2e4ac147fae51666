// Helpers shared by the marching kernels (K1 sweep, K2 residual+restriction).
#pragma once

#include <cuda_runtime.h>

#include "spaimg_common.cuh"

namespace spaimg {

template <class T, int S>
__device__ __forceinline__ int toff(const Terms<T>& M, int k, int a) {
    if constexpr (S == SHAPE_GENERIC) {
        return M.off[k][a];
    } else {
        return ShapeT<S>::o(k, a);
    }
}
template <class T, int S>
__device__ __forceinline__ int tnt(const Terms<T>& M) {
    if constexpr (S == SHAPE_GENERIC) {
        return M.nt;
    } else {
        return ShapeT<S>::nt;
    }
}

template <class T> struct V16;
template <> struct V16<double> {
    using type = double2;
    static __device__ __forceinline__ void ld(const double* p, double* v) {
        const double2 t = *reinterpret_cast<const double2*>(p);
        v[0] = t.x;
        v[1] = t.y;
    }
    static __device__ __forceinline__ void st(double* p, const double* v) {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    }
    // two consecutive elements (16 B for double)
    static __device__ __forceinline__ void ld2(const double* p, double* v) { ld(p, v); }
    static __device__ __forceinline__ void st2(double* p, const double* v) { st(p, v); }
};
template <> struct V16<float> {
    using type = float4;
    static __device__ __forceinline__ void ld(const float* p, float* v) {
        const float4 t = *reinterpret_cast<const float4*>(p);
        v[0] = t.x;
        v[1] = t.y;
        v[2] = t.z;
        v[3] = t.w;
    }
    static __device__ __forceinline__ void st(float* p, const float* v) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
    // two consecutive elements (8 B for float)
    static __device__ __forceinline__ void ld2(const float* p, float* v) {
        const float2 t = *reinterpret_cast<const float2*>(p);
        v[0] = t.x;
        v[1] = t.y;
    }
    static __device__ __forceinline__ void st2(float* p, const float* v) {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    }
};

// row-marching kernels: value of r row (o0 = -1, 0, +1 -> rm, rc, rp) at column v + o1 of this lane
template <class T, int VEC>
__device__ __forceinline__ T pick(const T* rm, const T* rc, const T* rp, T lm, T lc, T lp, T hm, T hc, T hp, int o0,
                                  int o1, int v) {
    const T* row = o0 < 0 ? rm : (o0 == 0 ? rc : rp);
    if (o1 == 0) return row[v];
    if (o1 < 0) return v > 0 ? row[v - 1] : (o0 < 0 ? lm : (o0 == 0 ? lc : lp));
    return v + 1 < VEC ? row[v + 1] : (o0 < 0 ? hm : (o0 == 0 ? hc : hp));
}

// streaming 16-byte global store that does not allocate in L1
template <class T>
__device__ __forceinline__ void stg16(T* p, const T* v) { V16<T>::st(p, v); }

// Flat tile kernels: stage r = b - A x (FZ: r = b, the iterate is zero) at CNT points of a tile
// footprint, NTH threads, in groups of BATCH points per thread whose global loads are all issued
// before the first use.  (The rolled per-point loop these kernels started with paid one L2 round
// trip per point: bounds branch, 6-8 dependent-on-nothing loads, arithmetic, store, next point.)
//   idx(q, p): footprint point q -> true and its element offset p when it is an interior point
//   put(q, r): store the residual of footprint point q (zero outside the interior)
// Out-of-range points load from the interior origin (always addressable) and discard the value.
template <class T, int D, bool FZ, int CNT, int NTH, int BATCH, class Idx, class Put>
__device__ __forceinline__ void flat_stage_r(const T* __restrict__ x, const T* __restrict__ b, const Layout& L, T sA,
                                             Idx idx, Put put) {
    constexpr int IT = (CNT + NTH - 1) / NTH;
    constexpr int NL = FZ ? 1 : (D == 2 ? 6 : 8);
#pragma unroll
    for (int i0 = 0; i0 < IT; i0 += BATCH) {
        T v[BATCH][NL];
        bool ok[BATCH];
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
            ok[u] = false;
            if (i0 + u < IT) {
                // branch-free: every load of the group must be issuable before the first use
                const int q = (i0 + u) * NTH + (int)threadIdx.x;
                long long p = L.origin;
                const bool in = idx(q, p);
                ok[u] = ((i0 + u + 1) * NTH <= CNT || q < CNT) & in;
                p = ok[u] ? p : L.origin;
                v[u][0] = b[p];
                if constexpr (!FZ) {
                    v[u][1] = x[p];
                    if constexpr (D == 2) {
                        v[u][2] = x[p + L.px];
                        v[u][3] = x[p - L.px];
                        v[u][4] = x[p + 1];
                        v[u][5] = x[p - 1];
                    } else {
                        v[u][2] = x[p + L.pp];
                        v[u][3] = x[p - L.pp];
                        v[u][4] = x[p + L.px];
                        v[u][5] = x[p - L.px];
                        v[u][6] = x[p + 1];
                        v[u][7] = x[p - 1];
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
            if (i0 + u < IT) {
                const int q = (i0 + u) * NTH + (int)threadIdx.x;
                T rv;
                if constexpr (FZ) {
                    rv = v[u][0];  // b - A 0 == b exactly
                } else if constexpr (D == 2) {
                    rv = residual2d<T>(v[u][0], v[u][1], v[u][2], v[u][3], v[u][4], v[u][5], sA);
                } else {
                    rv = residual3d<T>(v[u][0], v[u][1], v[u][2], v[u][3], v[u][4], v[u][5], v[u][6], v[u][7], sA);
                }
                rv = ok[u] ? rv : T(0);
                if ((i0 + u + 1) * NTH <= CNT || q < CNT) put(q, rv);
            }
        }
    }
}

// Chunk count along the marching axis for `tiles` CTAs per chunk row and `slots` resident CTA
// slots: favour a whole number of waves (a partial last wave leaves most SMs idle while a few
// CTAs march their whole chunk) while amortising each chunk's pipeline fill (`fill` extra
// rows/planes staged per chunk of `len`).
inline int march_chunks(int tiles, int slots, int span, int min_len, int fill) {
    int best = 1;
    double best_e = -1.0;
    for (int c = 1; c <= span; ++c) {
        const int len = (span + c - 1) / c;
        if (len < min_len && c > 1) break;
        const int cc = (span + len - 1) / len;
        const long long ctas = (long long)tiles * cc;
        const long long waves = (ctas + slots - 1) / slots;
        if (waves > 16) break;
        const double e = (double)ctas / (double)(waves * slots) * len / (double)(len + fill);
        if (e > best_e + 1e-9) {
            best_e = e;
            best = cc;
        }
    }
    return best;
}

inline int num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace spaimg

namespace spaimg {

// Deterministic residual-norm epilogue shared by the fused kernels: each CTA reduces its
// threads' partial sums of r^2 (fixed shuffle tree, fixed warp order), stores the CTA partial,
// and the last CTA to finish (atomic ticket) adds all partials in index order and appends
// sqrt(sum) to the device-side residual history at *slot (then advances *slot).  The result is
// independent of CTA scheduling; no floating-point atomics.


__device__ __forceinline__ void norm_epilogue(double s, const NormOut& no) {
    __shared__ double red[32];
    __shared__ bool last;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    const int nw = (blockDim.x + 31) >> 5;
    __syncthreads();
    if (l == 0) red[w] = s;
    __syncthreads();
    const unsigned nblocks = gridDim.x * gridDim.y * gridDim.z;
    const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < nw; ++i) t += red[i];
        no.partials[bid] = t;
        __threadfence();
        last = atomicAdd(no.counter, 1u) == nblocks - 1;
    }
    __syncthreads();
    if (last && w == 0) {
        __threadfence();
        double t = 0.0;
        for (unsigned i = l; i < nblocks; i += 32) t += ((volatile double*)no.partials)[i];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (l == 0) {
            const int sl = *no.slot;
            const double nrm = sqrt(t);
            no.norms[sl] = nrm;
            *no.slot = sl + 1;
            *no.counter = 0u;
            if (no.ctl) {  // k = sl cycles done; the k_solve_check logic
                const bool conv = sl >= 1 && nrm <= no.ctl->tol * no.norms[0];
                const bool cont = !conv && sl < no.ctl->max_iters;
                no.state[0] = sl;
                no.state[1] = conv ? 1 : 0;
                cudaGraphSetConditional(no.cond, cont ? 1u : 0u);
            }
        }
    }
}

}  // namespace spaimg
