// Device-side building blocks of the shared-memory coarse engine (K5+), shared by the generic
// op-list interpreter (kernels_tail.cu) and the compile-time recursion for power-of-two
// hierarchies (kernels_tail_fast.cuh): the point ops on one level held in shared memory, the
// coarse direct solves, the correctly rounded pivot division.  See kernels_tail.cu for the design.
#pragma once

#include "kernels.h"

namespace spaimg {

constexpr int NT = kTailThreads;

// ------------------------------------------------------------------------------------------
// division by a fixed pivot d with its precomputed correctly rounded reciprocal rcp = RN(1/d):
// q0 = y*rcp, then two Markstein corrections q += (y - d q) rcp.  After the first correction q
// is within one ulp of y/d, so the second returns RN(y/d) exactly (Markstein's theorem, given no
// underflow in y - d q); outside the guarded exponent range (and for 0, inf, nan) the plain
// IEEE division runs.  42 cycles of dependent latency instead of 125 for __ddiv_rn (measured,
// tools/dp_probe.cu), on the critical path of the coarse back substitution.
// ------------------------------------------------------------------------------------------
template <class T> __device__ __forceinline__ T pivot_div(T y, T d, T rcp);
template <> __device__ __forceinline__ double pivot_div<double>(double y, double d, double rcp) {
    const double ay = fabs(y);
    if (!(ay >= 0x1p-900 && ay <= 0x1p900)) return __ddiv_rn(y, d);
    double q = __dmul_rn(y, rcp);
    double r = __fma_rn(-d, q, y);
    q = __fma_rn(r, rcp, q);
    r = __fma_rn(-d, q, y);
    return __fma_rn(r, rcp, q);
}
template <> __device__ __forceinline__ float pivot_div<float>(float y, float d, float) { return __fdiv_rn(y, d); }

// ------------------------------------------------------------------------------------------
// stencil shapes as (d0, d1, d2) offsets, d0 along the strip axis 0, d2 the contiguous axis
// (2D: d1 == 0); which tile columns (d1, d2) a shape touches and the d0 range it needs there
// ------------------------------------------------------------------------------------------
template <int S, int D> struct Sh {
    static constexpr int nt = ShapeT<S>::nt;
    __host__ __device__ static constexpr int d0(int k) { return ShapeT<S>::o(k, 0); }
    __host__ __device__ static constexpr int d1(int k) { return D == 3 ? ShapeT<S>::o(k, 1) : 0; }
    __host__ __device__ static constexpr int d2(int k) { return D == 3 ? ShapeT<S>::o(k, 2) : ShapeT<S>::o(k, 1); }
    __host__ __device__ static constexpr bool used(int e1, int e2) {
        for (int k = 0; k < nt; ++k)
            if (d1(k) == e1 && d2(k) == e2) return true;
        return false;
    }
    __host__ __device__ static constexpr int lo(int e1, int e2) {
        int v = 2;
        for (int k = 0; k < nt; ++k)
            if (d1(k) == e1 && d2(k) == e2 && d0(k) < v) v = d0(k);
        return v;
    }
    __host__ __device__ static constexpr int hi(int e1, int e2) {
        int v = -2;
        for (int k = 0; k < nt; ++k)
            if (d1(k) == e1 && d2(k) == e2 && d0(k) > v) v = d0(k);
        return v;
    }
};
// the Laplacian's shape in each dimension (stencils.py:209-223 term order)
template <int D> constexpr int kLapShape = D == 2 ? SHAPE_STAR5 : SHAPE_STAR7;

// thread -> strip of a level's W^D box over NTH threads: K points along axis 0 at cross-section
// (i1, i2).  NTH = 512 (the CTA) for the big levels; NTH = 32 runs a small level in one warp.
template <int D, int LOGW, int NTH = NT> struct Strip {
    static constexpr int W = 1 << LOGW;
    static constexpr int PTS = D == 2 ? W * W : W * W * W;
    static constexpr int K = PTS > NTH ? PTS / NTH : 1;
    static constexpr int ACT = PTS / K;  // threads with a strip
    static constexpr int XS = (D - 1) * LOGW;
    int i0, i1, i2;  // first point of the strip
    bool ok;         // thread owns a strip whose cross-section is inside the interior
    __device__ __forceinline__ explicit Strip(int n) {
        const int t = threadIdx.x;
        const int c = t & ((1 << XS) - 1);
        i2 = c & (W - 1);
        i1 = D == 3 ? (c >> LOGW) : 0;
        i0 = (t >> XS) * K;
        ok = t < ACT && i2 < n && (D == 2 || i1 < n) && i0 < n;
    }
    __device__ __forceinline__ int at(int s0, int s1) const { return i0 * s0 + i1 * s1 + i2; }
};

// ------------------------------------------------------------------------------------------
// register tile of a shape around a strip: v[1 + j][1 + e1][1 + e2] = src[p0 + j s0 + e1 s1 + e2]
// for the rows j each used column needs (j in [lo, K - 1 + hi])
// ------------------------------------------------------------------------------------------
template <class T, int S, int D, int K> struct Tile {
    T v[K + 2][3][3];
    __device__ __forceinline__ void load(const T* src, int p0, int s0, int s1) {
        using H = Sh<S, D>;
#pragma unroll
        for (int e1 = -1; e1 <= 1; ++e1)
#pragma unroll
            for (int e2 = -1; e2 <= 1; ++e2) {
                if (!H::used(e1, e2)) continue;
#pragma unroll
                for (int j = H::lo(e1, e2); j <= K - 1 + H::hi(e1, e2); ++j)
                    v[1 + j][1 + e1][1 + e2] = src[p0 + j * s0 + e1 * s1 + e2];
            }
    }
    // term k of the shape at strip row j
    __device__ __forceinline__ T at(int j, int k) const {
        using H = Sh<S, D>;
        return v[1 + j + H::d0(k)][1 + H::d1(k)][1 + H::d2(k)];
    }
};

// ------------------------------------------------------------------------------------------
// point ops
// ------------------------------------------------------------------------------------------
template <class T, int D, int LOGW, int NTH = NT>
__device__ __forceinline__ void op_res(const TailLv<T>& f, T* arr) {
    using Q = Strip<D, LOGW, NTH>;
    const Q q(f.n);
    if (!q.ok) return;
    constexpr int K = Q::K;
    constexpr int LS = kLapShape<D>;
    const int s0 = f.s0, s1 = f.s1;
    const int p0 = q.at(s0, s1);
    const T* x = arr + f.x;
    const T* b = arr + f.b;
    T* r = arr + f.r;
    Tile<T, LS, D, K> X;
    X.load(x, p0, s0, s1);
    T bv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) bv[j] = b[p0 + j * s0];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (q.i0 + j >= f.n) break;
        T v;
        if constexpr (D == 2)
            v = residual2d<T>(bv[j], X.at(j, 0), X.at(j, 1), X.at(j, 2), X.at(j, 3), X.at(j, 4), f.sA);
        else
            v = residual3d<T>(bv[j], X.at(j, 0), X.at(j, 1), X.at(j, 2), X.at(j, 3), X.at(j, 4), X.at(j, 5), X.at(j, 6),
                              f.sA);
        r[p0 + j * s0] = v;
    }
}

// x = (FROM_ZERO ? 0 : x) + omega ((M src) sM) with src = r (RELAX) or b (RELAX0: r == b)
template <class T, int S, int D, int LOGW, bool FROM_ZERO, int NTH = NT>
__device__ __forceinline__ void op_relax(const TailLv<T>& f, T* arr, const Terms<T>& M, T omega) {
    using O = Op<T>;
    using Q = Strip<D, LOGW, NTH>;
    const Q q(f.n);
    if (!q.ok) return;
    constexpr int K = Q::K;
    const int s0 = f.s0, s1 = f.s1;
    const int p0 = q.at(s0, s1);
    const T* src = arr + (FROM_ZERO ? f.b : f.r);
    T* x = arr + f.x;
    T xv[K];
    if constexpr (!FROM_ZERO) {
#pragma unroll
        for (int j = 0; j < K; ++j) xv[j] = x[p0 + j * s0];
    }
    if constexpr (S == SHAPE_GENERIC) {
        T acc[K];
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = T(0);
        for (int k = 0; k < M.nt; ++k) {
            const int off = D == 2 ? M.off[k][0] * s0 + M.off[k][1] : M.off[k][0] * s0 + M.off[k][1] * s1 + M.off[k][2];
            const T c = M.c[k];
#pragma unroll
            for (int j = 0; j < K; ++j) acc[j] = O::add(acc[j], O::mul(c, src[p0 + j * s0 + off]));
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (q.i0 + j >= f.n) break;
            x[p0 + j * s0] = relax<T>(FROM_ZERO ? T(0) : xv[j], acc[j], f.sM, omega);
        }
    } else {
        Tile<T, S, D, K> R;
        R.load(src, p0, s0, s1);
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (q.i0 + j >= f.n) break;
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < Sh<S, D>::nt; ++k) acc = O::add(acc, O::mul(M.c[k], R.at(j, k)));
            x[p0 + j * s0] = relax<T>(FROM_ZERO ? T(0) : xv[j], acc, f.sM, omega);
        }
    }
}

template <class T, int D, int LOGW, int NTH = NT>
__device__ __forceinline__ void op_zero(const TailLv<T>& f, T* arr) {
    using Q = Strip<D, LOGW, NTH>;
    const Q q(f.n);
    if (!q.ok) return;
    const int p0 = q.at(f.s0, f.s1);
#pragma unroll
    for (int j = 0; j < Q::K; ++j)
        if (q.i0 + j < f.n) arr[f.x + p0 + j * f.s0] = T(0);
}

// coarse b = full weighting of the fine r (separable: axis 0, then 1, then 2; multigrid.py:104-119).
// LOGW is the FINE level's; the coarse points are mapped on the (W/2)^D box.
template <class T, int D, int LOGW, int NTH = NT>
__device__ __forceinline__ void op_fw(const TailLv<T>& f, const TailLv<T>& c, T* arr) {
    using Q = Strip<D, LOGW - 1, NTH>;
    const Q q(c.n);
    if (!q.ok) return;
    constexpr int K = Q::K;
    constexpr int E1 = D == 3 ? 3 : 1;
    const T* r = arr + f.r;
    T* bc = arr + c.b;
    const int s0 = f.s0, s1 = f.s1;
    // fine rows 2 i0 .. 2 (i0 + K - 1) + 2 of the 3^(D-1) fine columns under the coarse column
    const int f0 = (2 * q.i0) * s0 + (2 * q.i1) * s1 + 2 * q.i2;
    T F[2 * K + 1][E1][3];
#pragma unroll
    for (int j = 0; j < 2 * K + 1; ++j)
#pragma unroll
        for (int e1 = 0; e1 < E1; ++e1)
#pragma unroll
            for (int e2 = 0; e2 < 3; ++e2) F[j][e1][e2] = r[f0 + j * s0 + e1 * s1 + e2];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (q.i0 + j >= c.n) break;
        T v;
        if constexpr (D == 2) {
            T t[3];
#pragma unroll
            for (int e2 = 0; e2 < 3; ++e2) t[e2] = fw<T>(F[2 * j][0][e2], F[2 * j + 1][0][e2], F[2 * j + 2][0][e2]);
            v = fw<T>(t[0], t[1], t[2]);
        } else {
            T u[3];
#pragma unroll
            for (int e2 = 0; e2 < 3; ++e2) {
                T t[3];
#pragma unroll
                for (int e1 = 0; e1 < 3; ++e1)
                    t[e1] = fw<T>(F[2 * j][e1][e2], F[2 * j + 1][e1][e2], F[2 * j + 2][e1][e2]);
                u[e2] = fw<T>(t[0], t[1], t[2]);
            }
            v = fw<T>(u[0], u[1], u[2]);
        }
        bc[(q.i0 + j) * c.s0 + q.i1 * c.s1 + q.i2] = v;
    }
}

// the reference's even-index formula (pl_even: ends 0.5 a[0] / 0.5 a[m-1], else 0.5 (a[j-1] + a[j]))
// evaluated branch-free: all three candidates formed, one selected (bitwise the same value)
template <class T>
__device__ __forceinline__ T pl_sel(T am1, T a0, bool first, bool last) {
    using O = Op<T>;
    const T vf = O::mul(T(0.5), a0), vl = O::mul(T(0.5), am1), vm = O::mul(T(0.5), O::add(am1, a0));
    return first ? vf : (last ? vl : vm);
}
// interpolant at fine line index i from A = g(j - 1), B = g(j), j = i >> 1: odd i -> g((i-1)/2) = B
template <class T>
__device__ __forceinline__ T lin(int i, int m, T A, T B) {
    const int j = i >> 1;
    const T ev = pl_sel<T>(A, B, j == 0, j == m);
    return (i & 1) ? B : ev;
}

// x = x + P e, separable d-linear prolongation, axis 0 first (multigrid.py:122-144, :184).  Each
// fine point reads the 2^D coarse values around it (rows j-1, j of every axis; the zero frame
// stands in outside) and interpolates branch-free; a strip of K rows (K even, starting on an even
// row) shares its K/2 + 1 coarse rows.
template <class T, int D, int LOGW, int NTH = NT>
__device__ __forceinline__ void op_prolong(const TailLv<T>& f, const TailLv<T>& c, T* arr) {
    using O = Op<T>;
    using Q = Strip<D, LOGW, NTH>;
    const Q q(f.n);
    if (!q.ok) return;
    constexpr int K = Q::K;
    constexpr int NR = K == 1 ? 2 : K / 2 + 1;  // coarse rows of the strip
    constexpr int E1 = D == 3 ? 2 : 1;
    const int s0 = f.s0;
    const int p0 = q.at(s0, f.s1);
    T* x = arr + f.x;
    const T* e = arr + c.x;
    const int m = c.n, cs0 = c.s0, cs1 = c.s1;
    const int j1 = q.i1 >> 1, j2 = q.i2 >> 1;
    const int cb = (q.i0 >> 1) - 1;
    T E[NR][E1][2];
#pragma unroll
    for (int a = 0; a < NR; ++a)
#pragma unroll
        for (int b = 0; b < E1; ++b)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc)
                E[a][b][cc] = e[(cb + a) * cs0 + (D == 3 ? (j1 - 1 + b) * cs1 : 0) + (j2 - 1 + cc)];
    T xv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) xv[j] = x[p0 + j * s0];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (q.i0 + j >= f.n) break;
        const int i0 = q.i0 + j;
        const int ra = K == 1 ? 0 : (j >> 1);  // row of g(j0 - 1) in E
        T u[E1][2];
#pragma unroll
        for (int b = 0; b < E1; ++b)
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) u[b][cc] = lin<T>(i0, m, E[ra][b][cc], E[ra + 1][b][cc]);
        T v[2];
        if constexpr (D == 3) {
#pragma unroll
            for (int cc = 0; cc < 2; ++cc) v[cc] = lin<T>(q.i1, m, u[0][cc], u[1][cc]);
        } else {
            v[0] = u[0][0];
            v[1] = u[0][1];
        }
        x[p0 + j * s0] = O::add(xv[j], lin<T>(q.i2, m, v[0], v[1]));
    }
}

// ------------------------------------------------------------------------------------------
// fused small-level ops of the compile-time engine (one op, one barrier instead of two)
// ------------------------------------------------------------------------------------------
// coarse b = full weighting of r = b - A x, r formed on the fly at the 3^D fine points under each
// coarse point (multigrid.py:176-177); one coarse point per thread (K = 1 boxes only)
template <class T, int D, int LOGW, int NTH = NT>
__device__ __forceinline__ void op_resfw(const TailLv<T>& f, const TailLv<T>& c, T* arr) {
    using Q = Strip<D, LOGW - 1, NTH>;
    static_assert(Q::K == 1, "op_resfw maps one coarse point per thread");
    const Q q(c.n);
    if (!q.ok) return;
    const int s0 = f.s0, s1 = f.s1;
    const T* x = arr + f.x;
    const T* b = arr + f.b;
    const int f0 = (2 * q.i0) * s0 + (2 * q.i1) * s1 + 2 * q.i2;  // fine point (2I, 2J[, 2K])
    constexpr int E1 = D == 3 ? 3 : 1;
    T r[3][E1][3];
#pragma unroll
    for (int a0 = 0; a0 < 3; ++a0)
#pragma unroll
        for (int a1 = 0; a1 < E1; ++a1)
#pragma unroll
            for (int a2 = 0; a2 < 3; ++a2) {
                const int p = f0 + a0 * s0 + a1 * s1 + a2;
                if constexpr (D == 2)
                    r[a0][a1][a2] = residual2d<T>(b[p], x[p], x[p + s0], x[p - s0], x[p + 1], x[p - 1], f.sA);
                else
                    r[a0][a1][a2] = residual3d<T>(b[p], x[p], x[p + s0], x[p - s0], x[p + s1], x[p - s1], x[p + 1],
                                                  x[p - 1], f.sA);
            }
    T v;
    if constexpr (D == 2) {
        T t[3];
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) t[a2] = fw<T>(r[0][0][a2], r[1][0][a2], r[2][0][a2]);
        v = fw<T>(t[0], t[1], t[2]);
    } else {
        T u[3];
#pragma unroll
        for (int a2 = 0; a2 < 3; ++a2) {
            T t[3];
#pragma unroll
            for (int a1 = 0; a1 < 3; ++a1) t[a1] = fw<T>(r[0][a1][a2], r[1][a1][a2], r[2][a1][a2]);
            u[a2] = fw<T>(t[0], t[1], t[2]);
        }
        v = fw<T>(u[0], u[1], u[2]);
    }
    arr[c.b + q.i0 * c.s0 + q.i1 * c.s1 + q.i2] = v;
}

// ------------------------------------------------------------------------------------------
// coarse direct solve in getrs order (Appendix A.5/A.6): y = P b; column-oriented unit-lower
// forward substitution with FMA; column-oriented upper back substitution with a correctly
// rounded division.
// ------------------------------------------------------------------------------------------
// one thread, all unknowns in registers, the factors straight from the kernel parameters (NLU =
// 1, 9, 27: coarsest_N = 2 or 4).  Each unknown sees the updates of the sequential loops in the
// same j order.
template <class T, int NLU>
__device__ __forceinline__ void coarse_thread(const TailArgs<T>& a, const TailLv<T>& c, T* arr) {
    using O = Op<T>;
    if (threadIdx.x != 0) return;
    const T* b = arr + c.b;
    T* x = arr + c.x;
    T y[NLU];
#pragma unroll
    for (int i = 0; i < NLU; ++i) y[i] = b[a.cin[i]];
#pragma unroll
    for (int j = 0; j < NLU; ++j)
#pragma unroll
        for (int i = j + 1; i < NLU; ++i) y[i] = O::fma(a.lu[i * NLU + j], y[j], y[i]);
#pragma unroll
    for (int j = NLU - 1; j >= 0; --j) {
        y[j] = pivot_div<T>(y[j], a.dg[j], a.rc[j]);
#pragma unroll
        for (int i = 0; i < j; ++i) y[i] = O::fma(a.lu[i * NLU + j], y[j], y[i]);
    }
#pragma unroll
    for (int i = 0; i < NLU; ++i) x[a.cout[i]] = y[i];
}

// one warp, lane i holds y_i (other nlu <= 27; factors in the parameters)
template <class T>
__device__ __forceinline__ void coarse_warp(const TailArgs<T>& a, const TailLv<T>& c, T* arr) {
    using O = Op<T>;
    const int l = threadIdx.x, nlu = a.nlu;
    const T* b = arr + c.b;
    T* x = arr + c.x;
    T y = l < nlu ? b[a.cin[l]] : T(0);
    for (int j = 0; j < nlu; ++j) {
        const T yj = __shfl_sync(0xffffffffu, y, j);
        if (l > j && l < nlu) y = O::fma(a.lu[l * nlu + j], yj, y);
    }
    for (int j = nlu - 1; j >= 0; --j) {
        if (l == j) y = pivot_div<T>(y, a.dg[j], a.rc[j]);
        const T yj = __shfl_sync(0xffffffffu, y, j);
        if (l < j) y = O::fma(a.lu[l * nlu + j], yj, y);
    }
    if (l < nlu) x[a.cout[l]] = y;
}

// the whole CTA (nlu > kTailMaxLU): factors in shared memory (cf = [-LU | U_jj | 1/U_jj],
// ci = [b offsets | x offsets]), y in shared memory
template <class T>
__device__ __forceinline__ void coarse_block(const TailLv<T>& c, T* arr, const T* cf, const int* ci, int nlu, T* y) {
    using O = Op<T>;
    const T* b = arr + c.b;
    T* x = arr + c.x;
    for (int i = threadIdx.x; i < nlu; i += NT) y[i] = b[ci[i]];
    __syncthreads();
    for (int j = 0; j < nlu; ++j) {
        const T yj = y[j];
        for (int i = j + 1 + threadIdx.x; i < nlu; i += NT) y[i] = O::fma(cf[i * nlu + j], yj, y[i]);
        __syncthreads();
    }
    for (int j = nlu - 1; j >= 0; --j) {
        if (threadIdx.x == 0) y[j] = pivot_div<T>(y[j], cf[nlu * nlu + j], cf[nlu * nlu + nlu + j]);
        __syncthreads();
        const T yj = y[j];
        for (int i = threadIdx.x; i < j; i += NT) y[i] = O::fma(cf[i * nlu + j], yj, y[i]);
        __syncthreads();
    }
    for (int i = threadIdx.x; i < nlu; i += NT) x[ci[nlu + i]] = y[i];
}

// ------------------------------------------------------------------------------------------
// coarse solve for the compile-time engine: one thread, factors in shared memory
// (cf = [-LU off the diagonal, row-major | U_jj | 1/U_jj], ci = [b offsets | x offsets]).  The
// back substitution continues with the quotient after ONE Markstein correction (q1, 24 cycles
// after y_j is final instead of 40) and checks it against the correctly rounded q2 off the
// critical path; a system where any q1 != q2 (or a value outside the guarded range) is solved
// again with IEEE divisions -- the result is bitwise the exact-division result either way.
// ------------------------------------------------------------------------------------------
template <class T, int NLU>
__device__ __noinline__ void coarse_exact(const T* cf, const int* ci, const T* b, T* x) {
    using O = Op<T>;
    T y[NLU];
#pragma unroll
    for (int i = 0; i < NLU; ++i) y[i] = b[ci[i]];
#pragma unroll
    for (int j = 0; j < NLU; ++j)
#pragma unroll
        for (int i = j + 1; i < NLU; ++i) y[i] = O::fma(cf[i * NLU + j], y[j], y[i]);
#pragma unroll
    for (int j = NLU - 1; j >= 0; --j) {
        y[j] = O::div(y[j], cf[NLU * NLU + j]);
#pragma unroll
        for (int i = 0; i < j; ++i) y[i] = O::fma(cf[i * NLU + j], y[j], y[i]);
    }
#pragma unroll
    for (int i = 0; i < NLU; ++i) x[ci[NLU + i]] = y[i];
}

template <class T, int NLU>
__device__ __forceinline__ void coarse_fast(const T* cf, const int* ci, const T* b, T* x) {
    using O = Op<T>;
    T y[NLU];
#pragma unroll
    for (int i = 0; i < NLU; ++i) y[i] = b[ci[i]];
#pragma unroll
    for (int j = 0; j < NLU; ++j)
#pragma unroll
        for (int i = j + 1; i < NLU; ++i) y[i] = O::fma(cf[i * NLU + j], y[j], y[i]);
    bool ok = true;
#pragma unroll
    for (int j = NLU - 1; j >= 0; --j) {
        if constexpr (sizeof(T) == 8) {
            const T v = y[j], d = cf[NLU * NLU + j], rcp = cf[NLU * NLU + NLU + j];
            const double av = fabs(v);
            const T q0 = O::mul(v, rcp);
            const T q1 = O::fma(O::fma(-d, q0, v), rcp, q0);
            const T q2 = O::fma(O::fma(-d, q1, v), rcp, q1);
            ok = ok && av >= 0x1p-900 && av <= 0x1p900 && q2 == q1;
            y[j] = q1;
        } else {
            y[j] = O::div(y[j], cf[NLU * NLU + j]);
        }
#pragma unroll
        for (int i = 0; i < j; ++i) y[i] = O::fma(cf[i * NLU + j], y[j], y[i]);
    }
    if (!ok) {
        coarse_exact<T, NLU>(cf, ci, b, x);
        return;
    }
#pragma unroll
    for (int i = 0; i < NLU; ++i) x[ci[NLU + i]] = y[i];
}

// checked build: NaN on the interior of one shared-memory level array (origin offset `at`,
// interior n^D, frame F left at zero); at < 0 skips
template <class T, int D>
__device__ __forceinline__ void tail_poison(T* arr, int n, int F, int s0, int s1, int at) {
    if (at < 0) return;
    const int cnt = D == 2 ? n * n : n * n * n;
    for (int q = threadIdx.x; q < cnt; q += NT) {
        const int i0 = D == 2 ? q / n : q / (n * n);
        const int rem = D == 2 ? q - i0 * n : q - i0 * n * n;
        const int i1 = D == 2 ? 0 : rem / n;
        const int i2 = D == 2 ? rem : rem - i1 * n;
        arr[at + i0 * s0 + i1 * s1 + i2] = T(__int_as_float(0x7fc00000));
    }
}

// ------------------------------------------------------------------------------------------
// entry level: global padded layout <-> shared memory (frame F, pitches s0, s1)
// ------------------------------------------------------------------------------------------
// x and b: the box [-F, n+F)^D of the global padded layout, whose frame is zero, so the shared
// frames come out zero as well
template <class T, int D>
__device__ __forceinline__ void tail_load_entry(const TailArgs<T>& a, T* arr, int ex, int eb, int es0, int es1) {
    const int F = a.frame, n = a.gL.n, w = n + 2 * F;
    const int cnt = D == 2 ? w * w : w * w * w;
    for (int qq = threadIdx.x; qq < cnt; qq += NT) {
        int j0, j1, j2;
        if (D == 2) {
            j0 = qq / w;
            j1 = 0;
            j2 = qq - j0 * w;
        } else {
            j0 = qq / (w * w);
            const int rem = qq - j0 * w * w;
            j1 = rem / w;
            j2 = rem - j1 * w;
            j1 -= F;
        }
        j0 -= F;
        j2 -= F;
        const long long g = a.gL.origin + (long long)j0 * (D == 2 ? a.gL.px : a.gL.pp) +
                            (D == 3 ? (long long)j1 * a.gL.px : 0LL) + j2;
        const int s = j0 * es0 + j1 * es1 + j2;
        arr[eb + s] = a.gb[g];
        arr[ex + s] = a.gx[g];
    }
}

// the entry level's iterate (interior) back to global memory
template <class T, int D>
__device__ __forceinline__ void tail_store_entry(const TailArgs<T>& a, const T* arr, int ex, int es0, int es1) {
    const int n = a.gL.n;
    const int cnt = D == 2 ? n * n : n * n * n;
    for (int qq = threadIdx.x; qq < cnt; qq += NT) {
        int j0, j1, j2;
        if (D == 2) {
            j0 = qq / n;
            j1 = 0;
            j2 = qq - j0 * n;
        } else {
            j0 = qq / (n * n);
            const int rem = qq - j0 * n * n;
            j1 = rem / n;
            j2 = rem - j1 * n;
        }
        const long long g = a.gL.origin + (long long)j0 * (D == 2 ? a.gL.px : a.gL.pp) +
                            (D == 3 ? (long long)j1 * a.gL.px : 0LL) + j2;
        a.gx[g] = arr[ex + j0 * es0 + j1 * es1 + j2];
    }
}

}  // namespace spaimg
