// K5+: the shared-memory coarse-grid engine.  All levels from a size threshold down (2D n <= 63,
// 3D n <= 15) live in ONE CTA's shared memory, and the CTA runs the whole V/W recursion below
// its entry level (reference multigrid.py:157-185) without leaving the SM:
//   1. load the host-recorded op list and the coarse LU data into shared memory, copy the entry
//      level's b and start iterate (with their zero frames) from global memory, zero the rest;
//   2. interpret the ops, each point-parallel over its level; consecutive ops are separated by a
//      barrier over only the warps involved (__syncwarp for one warp, a named barrier per
//      distinct warp count, __syncthreads for all) -- the small levels of a W-cycle run on one
//      or two warps and do not pay for a 16-warp barrier;
//   3. store the entry level's iterate back to global memory (in place).
// Point mapping: a level's interior is embedded in a W^dim box (W = 1 << logw >= n); thread t
// owns one position of the box's (dim-1)-dimensional cross-section and a strip of K consecutive
// points along axis 0 (K = W^dim / 512 for the big levels, else 1), so a stencil's loads along
// axis 0 are shared between the strip's points (register tile) instead of re-read from shared
// memory (shared-memory bandwidth, 128 B/clk/SM, bounds the big levels).
// Every per-point expression is the Appendix-A tree of the multi-kernel path
// (spaimg_common.cuh), so the engine is bitwise identical to it; only the memory changes.  The
// relaxation updates x in place: x' at a point reads x only at that point (multigrid.py:100).
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

// thread -> strip of a level's W^D box: K points along axis 0 at cross-section (i1, i2)
template <int D, int LOGW> struct Strip {
    static constexpr int W = 1 << LOGW;
    static constexpr int PTS = D == 2 ? W * W : W * W * W;
    static constexpr int K = PTS > NT ? PTS / NT : 1;
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
template <class T, int D, int LOGW>
__device__ __forceinline__ void op_res(const TailOp<T>& o, T* arr) {
    using Q = Strip<D, LOGW>;
    const Q q(o.n);
    if (!q.ok) return;
    constexpr int K = Q::K;
    constexpr int LS = kLapShape<D>;
    const int p0 = q.at(o.s0, o.s1);
    const T* x = arr + o.a0;
    const T* b = arr + o.a1;
    T* r = arr + o.a2;
    Tile<T, LS, D, K> X;
    X.load(x, p0, o.s0, o.s1);
    T bv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) bv[j] = b[p0 + j * o.s0];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (q.i0 + j >= o.n) break;
        T v;
        if constexpr (D == 2)
            v = residual2d<T>(bv[j], X.at(j, 0), X.at(j, 1), X.at(j, 2), X.at(j, 3), X.at(j, 4), o.s);
        else
            v = residual3d<T>(bv[j], X.at(j, 0), X.at(j, 1), X.at(j, 2), X.at(j, 3), X.at(j, 4), X.at(j, 5), X.at(j, 6),
                              o.s);
        r[p0 + j * o.s0] = v;
    }
}

// x = (FROM_ZERO ? 0 : x) + omega ((M src) sM) with src = r (RELAX) or b (RELAX0: r == b)
template <class T, int S, int D, int LOGW, bool FROM_ZERO>
__device__ __forceinline__ void op_relax(const TailOp<T>& o, T* arr, const Terms<T>& M, T omega) {
    using O = Op<T>;
    using Q = Strip<D, LOGW>;
    const Q q(o.n);
    if (!q.ok) return;
    constexpr int K = Q::K;
    const int p0 = q.at(o.s0, o.s1);
    const T* src = arr + (FROM_ZERO ? o.a1 : o.a2);
    T* x = arr + o.a0;
    T xv[K];
    if constexpr (!FROM_ZERO) {
#pragma unroll
        for (int j = 0; j < K; ++j) xv[j] = x[p0 + j * o.s0];
    }
    if constexpr (S == SHAPE_GENERIC) {
        T acc[K];
#pragma unroll
        for (int j = 0; j < K; ++j) acc[j] = T(0);
        for (int k = 0; k < M.nt; ++k) {
            const int off = D == 2 ? M.off[k][0] * o.s0 + M.off[k][1]
                                   : M.off[k][0] * o.s0 + M.off[k][1] * o.s1 + M.off[k][2];
            const T c = M.c[k];
#pragma unroll
            for (int j = 0; j < K; ++j) acc[j] = O::add(acc[j], O::mul(c, src[p0 + j * o.s0 + off]));
        }
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (q.i0 + j >= o.n) break;
            x[p0 + j * o.s0] = relax<T>(FROM_ZERO ? T(0) : xv[j], acc[j], o.s, omega);
        }
    } else {
        Tile<T, S, D, K> R;
        R.load(src, p0, o.s0, o.s1);
#pragma unroll
        for (int j = 0; j < K; ++j) {
            if (q.i0 + j >= o.n) break;
            T acc = T(0);
#pragma unroll
            for (int k = 0; k < Sh<S, D>::nt; ++k) acc = O::add(acc, O::mul(M.c[k], R.at(j, k)));
            x[p0 + j * o.s0] = relax<T>(FROM_ZERO ? T(0) : xv[j], acc, o.s, omega);
        }
    }
}

template <class T, int D, int LOGW>
__device__ __forceinline__ void op_zero(const TailOp<T>& o, T* arr) {
    using Q = Strip<D, LOGW>;
    const Q q(o.n);
    if (!q.ok) return;
    const int p0 = q.at(o.s0, o.s1);
#pragma unroll
    for (int j = 0; j < Q::K; ++j)
        if (q.i0 + j < o.n) arr[o.a0 + p0 + j * o.s0] = T(0);
}

// coarse b = full weighting of the fine r (separable: axis 0, then 1, then 2; multigrid.py:104-119).
// LOGW is the FINE level's; the coarse points are mapped on the (W/2)^D box.
template <class T, int D, int LOGW>
__device__ __forceinline__ void op_fw(const TailOp<T>& o, T* arr) {
    using Q = Strip<D, LOGW - 1>;
    const Q q(o.m);
    if (!q.ok) return;
    constexpr int K = Q::K;
    constexpr int E1 = D == 3 ? 3 : 1;
    const T* r = arr + o.a2;
    T* bc = arr + o.a1;
    // fine rows 2 i0 .. 2 (i0 + K - 1) + 2 of the 3^(D-1) fine columns under the coarse column
    const int f0 = (2 * q.i0) * o.s0 + (2 * q.i1) * o.s1 + 2 * q.i2;
    T F[2 * K + 1][E1][3];
#pragma unroll
    for (int j = 0; j < 2 * K + 1; ++j)
#pragma unroll
        for (int e1 = 0; e1 < E1; ++e1)
#pragma unroll
            for (int e2 = 0; e2 < 3; ++e2) F[j][e1][e2] = r[f0 + j * o.s0 + e1 * o.s1 + e2];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (q.i0 + j >= o.m) break;
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
        bc[(q.i0 + j) * o.cs0 + q.i1 * o.cs1 + q.i2] = v;
    }
}

// interpolant of fine line index i from a coarse line accessor g(j) (zero frame outside):
// odd i = 2j+1 -> g(j); even i = 2j -> pl_even(g(j-1), g(j)) with the reference end formulas
template <class T, class G>
__device__ __forceinline__ T interp(int i, int m, G&& g) {
    if (i & 1) return g((i - 1) >> 1);
    const int j = i >> 1;
    return pl_even<T>(g(j - 1), g(j), j == 0, j == m);
}

// x = x + P e, separable d-linear prolongation, axis 0 first (multigrid.py:122-144, :184)
template <class T, int D, int LOGW>
__device__ __forceinline__ void op_prolong(const TailOp<T>& o, T* arr) {
    using O = Op<T>;
    using Q = Strip<D, LOGW>;
    const Q q(o.n);
    if (!q.ok) return;
    constexpr int K = Q::K;
    const int p0 = q.at(o.s0, o.s1);
    T* x = arr + o.a0;
    const T* e = arr + o.a1;
    const int m = o.m;
    T xv[K], pv[K];
#pragma unroll
    for (int j = 0; j < K; ++j) xv[j] = x[p0 + j * o.s0];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        const int i0 = q.i0 + j;
        if constexpr (D == 2) {
            auto t0 = [&](int j1) { return interp<T>(i0, m, [&](int j0) { return e[j0 * o.cs0 + j1]; }); };
            pv[j] = interp<T>(q.i2, m, t0);
        } else {
            auto t1 = [&](int j2) {
                auto t0 = [&](int j1) {
                    return interp<T>(i0, m, [&](int j0) { return e[j0 * o.cs0 + j1 * o.cs1 + j2]; });
                };
                return interp<T>(q.i1, m, t0);
            };
            pv[j] = interp<T>(q.i2, m, t1);
        }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
        if (q.i0 + j >= o.n) break;
        x[p0 + j * o.s0] = O::add(xv[j], pv[j]);
    }
}

// ------------------------------------------------------------------------------------------
// coarse direct solve in getrs order (Appendix A.5/A.6): y = P b; column-oriented unit-lower
// forward substitution with FMA; column-oriented upper back substitution with a correctly
// rounded division.  cf = [-LU off the diagonal | U_jj | 1/U_jj]; ci = [b offsets of the
// permuted rows | x offsets].
// ------------------------------------------------------------------------------------------
// one thread, all unknowns in registers (NLU = 1, 9, 27: coarsest_N = 2 or 4)
template <class T, int NLU>
__device__ __forceinline__ void coarse_thread(const TailOp<T>& o, T* arr, const T* cf, const int* ci) {
    using O = Op<T>;
    if (threadIdx.x != 0) return;
    const T* b = arr + o.a1;
    T* x = arr + o.a0;
    T y[NLU];
#pragma unroll
    for (int i = 0; i < NLU; ++i) y[i] = b[ci[i]];
#pragma unroll
    for (int j = 0; j < NLU; ++j)
#pragma unroll
        for (int i = j + 1; i < NLU; ++i) y[i] = O::fma(cf[i * NLU + j], y[j], y[i]);
#pragma unroll
    for (int j = NLU - 1; j >= 0; --j) {
        y[j] = pivot_div<T>(y[j], cf[NLU * NLU + j], cf[NLU * NLU + NLU + j]);
#pragma unroll
        for (int i = 0; i < j; ++i) y[i] = O::fma(cf[i * NLU + j], y[j], y[i]);
    }
#pragma unroll
    for (int i = 0; i < NLU; ++i) x[ci[NLU + i]] = y[i];
}

// one warp, lane i holds y_i (nlu <= 32)
template <class T>
__device__ __forceinline__ void coarse_warp(const TailOp<T>& o, T* arr, const T* cf, const int* ci, int nlu) {
    using O = Op<T>;
    const int l = threadIdx.x;
    const T* b = arr + o.a1;
    T* x = arr + o.a0;
    T y = l < nlu ? b[ci[l]] : T(0);
    for (int j = 0; j < nlu; ++j) {
        const T yj = __shfl_sync(0xffffffffu, y, j);
        if (l > j && l < nlu) y = O::fma(cf[l * nlu + j], yj, y);
    }
    for (int j = nlu - 1; j >= 0; --j) {
        if (l == j) y = pivot_div<T>(y, cf[nlu * nlu + j], cf[nlu * nlu + nlu + j]);
        const T yj = __shfl_sync(0xffffffffu, y, j);
        if (l < j) y = O::fma(cf[l * nlu + j], yj, y);
    }
    if (l < nlu) x[ci[nlu + l]] = y;
}

// the whole CTA, y in shared memory (nlu > 32)
template <class T>
__device__ __forceinline__ void coarse_block(const TailOp<T>& o, T* arr, const T* cf, const int* ci, int nlu, T* y) {
    using O = Op<T>;
    const T* b = arr + o.a1;
    T* x = arr + o.a0;
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
// the engine
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tail_barrier(int bid, int bw) {
    if (bid == 0) {
        __syncthreads();
    } else if (bid < 0) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(bid), "r"(bw * 32) : "memory");
    }
}

template <class T, int S, int D, int LOGW>
__device__ __forceinline__ void run_point_op(const TailOp<T>& o, T* arr, const Terms<T>& M, T omega) {
    switch (o.type) {
        case TAIL_RES: op_res<T, D, LOGW>(o, arr); break;
        case TAIL_RELAX: op_relax<T, S, D, LOGW, false>(o, arr, M, omega); break;
        case TAIL_RELAX0: op_relax<T, S, D, LOGW, true>(o, arr, M, omega); break;
        case TAIL_ZERO: op_zero<T, D, LOGW>(o, arr); break;
        case TAIL_FW: op_fw<T, D, LOGW>(o, arr); break;
        case TAIL_PROLONG: op_prolong<T, D, LOGW>(o, arr); break;
        default: break;
    }
}

template <class T, int S, int D>
__global__ void __launch_bounds__(NT, 1) k_tail(const TailArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    TailOp<T>* ops = reinterpret_cast<TailOp<T>*>(smem);
    T* cf = reinterpret_cast<T*>(smem + a.coarse_off);
    const int nlu = a.nlu;
    int* ci = reinterpret_cast<int*>(cf + nlu * nlu + 2 * nlu);
    T* arr = reinterpret_cast<T*>(smem + a.arr_off);
    T* ywork = arr + a.arr_elems;  // coarse_block's vector (nlu > 32 only)
    const int t = threadIdx.x;

    // 1. ops, coarse data, the entry level (frames included), zeroed scratch
    {
        const int4* src = reinterpret_cast<const int4*>(a.ops);
        int4* dst = reinterpret_cast<int4*>(ops);
        const int n16 = a.nops * (int)(sizeof(TailOp<T>) / 16);
        for (int i = t; i < n16; i += NT) dst[i] = src[i];
        const int ncf = nlu * nlu + 2 * nlu;
        for (int i = t; i < ncf; i += NT) cf[i] = a.coarse[i];
        for (int i = t; i < 2 * nlu; i += NT) ci[i] = a.coarse_idx[i];
        // entry level x and b: the box [-F, n+F)^D of the global padded layout, whose frame is
        // zero, so the shared frames come out zero as well
        const int F = a.frame, n = a.gL.n, w = n + 2 * F;
        const int cnt = D == 2 ? w * w : w * w * w;
        for (int qq = t; qq < cnt; qq += NT) {
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
            const int s = j0 * a.e_s0 + j1 * a.e_s1 + j2;
            arr[a.e_b + s] = a.gb[g];
            arr[a.e_x + s] = a.gx[g];
        }
        for (int i = a.zero_from + t; i < a.arr_elems; i += NT) arr[i] = T(0);
    }
    __syncthreads();

    // 2. the op list; op i+1 is fetched while op i runs
    const int warp = t >> 5;
    TailOp<T> op = ops[0];
    for (int i = 0; i < a.nops; ++i) {
        const TailOp<T> nxt = ops[i + 1 < a.nops ? i + 1 : i];
        if (warp < op.bw) {
            if (i > 0) tail_barrier(op.bid, op.bw);
            if (warp < op.nw) {
                if (op.type == TAIL_COARSE) {
                    if (nlu == 1)
                        coarse_thread<T, 1>(op, arr, cf, ci);
                    else if (nlu == 9)
                        coarse_thread<T, 9>(op, arr, cf, ci);
                    else if (nlu == 27)
                        coarse_thread<T, 27>(op, arr, cf, ci);
                    else if (nlu <= 32)
                        coarse_warp<T>(op, arr, cf, ci, nlu);
                    else
                        coarse_block<T>(op, arr, cf, ci, nlu, ywork);
                } else if (D == 2) {
                    switch (op.logw) {
                        case 2: run_point_op<T, S, D, 2>(op, arr, a.M, a.omega); break;
                        case 3: run_point_op<T, S, D, 3>(op, arr, a.M, a.omega); break;
                        case 4: run_point_op<T, S, D, 4>(op, arr, a.M, a.omega); break;
                        case 5: run_point_op<T, S, D, 5>(op, arr, a.M, a.omega); break;
                        case 6: run_point_op<T, S, D, 6>(op, arr, a.M, a.omega); break;
                        default: break;
                    }
                } else {
                    switch (op.logw) {
                        case 2: run_point_op<T, S, D, 2>(op, arr, a.M, a.omega); break;
                        case 3: run_point_op<T, S, D, 3>(op, arr, a.M, a.omega); break;
                        case 4: run_point_op<T, S, D, 4>(op, arr, a.M, a.omega); break;
                        default: break;
                    }
                }
            }
        }
        op = nxt;
    }
    __syncthreads();

    // 3. the entry level's iterate back to global memory (interior only)
    {
        const int n = a.gL.n;
        const int cnt = D == 2 ? n * n : n * n * n;
        for (int qq = t; qq < cnt; qq += NT) {
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
            a.gx[g] = arr[a.e_x + j0 * a.e_s0 + j1 * a.e_s1 + j2];
        }
    }
}

template <class T, int S, int D>
static cudaError_t launch_tail_s(const TailArgs<T>& a, cudaStream_t s) {
    if (a.smem > 48 * 1024) {  // per device, so set on every launch (host-side, cheap)
        cudaError_t e = cudaFuncSetAttribute(k_tail<T, S, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem);
        if (e != cudaSuccess) return e;
    }
    return launch_k(k_tail<T, S, D>, dim3(1), dim3(NT), a.smem, s, a);
}

template <class T>
cudaError_t launch_tail(const TailArgs<T>& a, cudaStream_t s) {
    if (a.gL.dim == 2) {
        switch (a.shape) {
            case SHAPE_C1: return launch_tail_s<T, SHAPE_C1, 2>(a, s);
            case SHAPE_STAR5: return launch_tail_s<T, SHAPE_STAR5, 2>(a, s);
            case SHAPE_BOX9: return launch_tail_s<T, SHAPE_BOX9, 2>(a, s);
            default: return launch_tail_s<T, SHAPE_GENERIC, 2>(a, s);
        }
    }
    switch (a.shape) {
        case SHAPE_C1: return launch_tail_s<T, SHAPE_C1, 3>(a, s);
        case SHAPE_STAR7: return launch_tail_s<T, SHAPE_STAR7, 3>(a, s);
        default: return launch_tail_s<T, SHAPE_GENERIC, 3>(a, s);
    }
}

template cudaError_t launch_tail<double>(const TailArgs<double>&, cudaStream_t);
template cudaError_t launch_tail<float>(const TailArgs<float>&, cudaStream_t);

}  // namespace spaimg
