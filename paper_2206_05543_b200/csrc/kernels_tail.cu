// K5+: single-block, shared-memory-resident tail of the cycle.  Every operation of the V/W
// recursion (reference multigrid.py:157-185) on the levels at or below a size threshold --
// smoothing sweeps, residual + restriction, the coarse direct solve, prolongation + correction
// -- runs inside ONE CTA of 1024 threads, instead of ~4 dependent graph nodes per level (each
// several microseconds of launch + memory latency for well under a microsecond of work).
//
// The host walks the same recursion as the multi-kernel schedule and records it as a list of
// TailOps.  The kernel
//   1. copies the op list and the level descriptors into shared memory,
//   2. zeroes the tail levels' compact shared-memory arrays (frame F = stencil radius: the
//      zero frame is the reference's zero extension, stencils.py:139-146),
//   3. loads the entry level's b (and x unless the entry starts from zero) from its global
//      level buffers,
//   4. interprets the ops, phases separated by __syncthreads(),
//   5. stores the entry level's resulting x back to its global buffer (the caller's
//      prolongation reads it there).
// Every per-point expression is the Appendix-A tree of the multi-kernel path
// (spaimg_common.cuh), so the tail is bitwise identical to it; only the memory changes.
#include <cstdlib>

#include "kernels.h"
#include "march.cuh"

namespace spaimg {

constexpr int kTailThreads = 1024;

// Tail levels are small (they fit one CTA's shared memory), so indices are 32-bit and the
// point -> (i0, i1[, i2]) split uses one approximate reciprocal instead of the integer division
// sequence (the largest stall source of the tail in the ncu source view).  tdiv(q, d) is exact
// for the tail's sizes: (q + 0.5)/d lies at least 0.5/d from an integer, and __fdividef's error
// (2 ulp of a quotient below n) stays under that for n*d < 2^20 (2D: n < 1024; 3D: n < 101).
__device__ __forceinline__ int tdiv(int q, int d) { return __float2int_rz(__fdividef((float)q + 0.5f, (float)d)); }

__device__ __forceinline__ int tidx(const Layout& L, int i0, int i1, int i2) {
    return (int)L.origin + i0 * (int)(L.dim == 2 ? L.px : L.pp) + (L.dim == 2 ? i1 : i1 * (int)L.px + i2);
}

// exact 64-bit versions for the cluster tail, whose levels live in global memory at any size
__device__ __forceinline__ long long gidx(const Layout& L, int i0, int i1, int i2) {
    return L.origin + (long long)i0 * (L.dim == 2 ? L.px : L.pp) + (L.dim == 2 ? (long long)i1 : (long long)i1 * L.px + i2);
}
__device__ __forceinline__ long long gpoint(const Layout& L, int q) {
    const int n = L.n;
    if (L.dim == 2) return L.origin + (long long)(q / n) * L.px + (q % n);
    const int i0 = q / (n * n), rem = q - i0 * n * n;
    return L.origin + (long long)i0 * L.pp + (long long)(rem / n) * L.px + (rem % n);
}

// interior point q (C order) -> padded index
__device__ __forceinline__ int tpoint(const Layout& L, int q) {
    const int n = L.n;
    if (L.dim == 2) {
        const int i0 = tdiv(q, n);
        return (int)L.origin + i0 * (int)L.px + (q - i0 * n);
    }
    const int i0 = tdiv(q, n * n), rem = q - i0 * n * n;
    const int i1 = tdiv(rem, n);
    return (int)L.origin + i0 * (int)L.pp + i1 * (int)L.px + (rem - i1 * n);
}

__device__ __forceinline__ int npoints(const Layout& L) { return L.dim == 2 ? L.n * L.n : L.n * L.n * L.n; }

template <class T>
__device__ __forceinline__ T tail_residual(const Layout& L, const T* x, const T* b, int p, T sA) {
    if (L.dim == 2) return residual2d<T>(b[p], x[p], x[p + L.px], x[p - L.px], x[p + 1], x[p - 1], sA);
    return residual3d<T>(b[p], x[p], x[p + L.pp], x[p - L.pp], x[p + L.px], x[p - L.px], x[p + 1], x[p - 1], sA);
}

// r = b - A x on every interior point (r = b exactly when x == 0, i.e. fz)
template <class T>
__device__ void tail_residual_phase(const TailLevel<T>& v, const T* x, bool fz) {
    const Layout& L = v.L;
    const int cnt = npoints(L);
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        const int p = tpoint(L, q);
        v.r[p] = fz ? v.b[p] : tail_residual<T>(L, x, v.b, p, v.sA);
    }
}

// xo = x + omega * ((M r) * sM)   (x == nullptr: from zero).  Named shapes (S != GENERIC) unroll
// the term loop with compile-time offsets, so every r load of a point issues at once.
template <class T, int S>
__device__ void tail_relax_phase(const TailLevel<T>& v, const T* x, T* xo, const Terms<T>& M, T omega) {
    using O = Op<T>;
    const Layout& L = v.L;
    const int cnt = npoints(L);
    const int px = (int)L.px, pp = (int)L.pp;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        const int p = tpoint(L, q);
        T acc = T(0);
        if constexpr (S == SHAPE_GENERIC) {
            for (int k = 0; k < M.nt; ++k) {
                const int o = L.dim == 2 ? M.off[k][0] * px + M.off[k][1]
                                         : M.off[k][0] * pp + M.off[k][1] * px + M.off[k][2];
                acc = O::add(acc, O::mul(M.c[k], v.r[p + o]));
            }
        } else {
            constexpr int NT = ShapeT<S>::nt;
            constexpr bool D3 = S == SHAPE_STAR7;
            T rv[NT];
#pragma unroll
            for (int k = 0; k < NT; ++k) {
                const int o = D3 ? ShapeT<S>::o(k, 0) * pp + ShapeT<S>::o(k, 1) * px + ShapeT<S>::o(k, 2)
                                 : ShapeT<S>::o(k, 0) * px + ShapeT<S>::o(k, 1);
                rv[k] = v.r[p + o];
            }
#pragma unroll
            for (int k = 0; k < NT; ++k) acc = O::add(acc, O::mul(M.c[k], rv[k]));
        }
        xo[p] = relax<T>(x ? x[p] : T(0), acc, v.sM, omega);
    }
}

// coarse right-hand side = full weighting of the fine residual (separable, axis 0 first)
template <class T>
__device__ void tail_restrict_phase(const TailLevel<T>& f, const TailLevel<T>& c) {
    const Layout& Lf = f.L;
    const Layout& Lc = c.L;
    const int m = Lc.n;
    const int cnt = npoints(Lc);
    const T* r = f.r;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        if (Lf.dim == 2) {
            const int I = tdiv(q, m), K = q - I * m;
            T t[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int p = tidx(Lf, 2 * I + 1, 2 * K + a, 0);
                t[a] = fw<T>(r[p - Lf.px], r[p], r[p + Lf.px]);
            }
            c.b[tidx(Lc, I, K, 0)] = fw<T>(t[0], t[1], t[2]);
        } else {
            const int I = tdiv(q, m * m), rem = q - I * m * m, J = tdiv(rem, m), K = rem - J * m;
            T u[3];
#pragma unroll
            for (int qk = 0; qk < 3; ++qk) {
                T t[3];
#pragma unroll
                for (int qj = 0; qj < 3; ++qj) {
                    const int p = tidx(Lf, 2 * I + 1, 2 * J + qj, 2 * K + qk);
                    t[qj] = fw<T>(r[p - Lf.pp], r[p], r[p + Lf.pp]);
                }
                u[qk] = fw<T>(t[0], t[1], t[2]);
            }
            c.b[tidx(Lc, I, J, K)] = fw<T>(u[0], u[1], u[2]);
        }
    }
}

// interpolant of fine line index i from a coarse line accessor g(j) (zero frame outside):
// odd i = 2j+1 -> g(j); even i = 2j -> pl_even(g(j-1), g(j)) with the reference end formulas
template <class T, class G>
__device__ __forceinline__ T tail_interp(int i, int m, G&& g) {
    if (i & 1) return g((i - 1) >> 1);
    const int j = i >> 1;
    return pl_even<T>(g(j - 1), g(j), j == 0, j == m);
}

// xo = xi + P e  (separable d-linear prolongation, axis 0 first; in place allowed)
template <class T>
__device__ void tail_prolong_phase(const TailLevel<T>& f, const TailLevel<T>& c, const T* xi, T* xo, const T* e) {
    using O = Op<T>;
    const Layout& Lf = f.L;
    const Layout& Lc = c.L;
    const int m = Lc.n;
    const int cnt = npoints(Lf);
    const int n = Lf.n;
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        T val;
        int p;
        if (Lf.dim == 2) {
            const int i0 = tdiv(q, n), i1 = q - i0 * n;
            p = tidx(Lf, i0, i1, 0);
            // axis 0 at fine row i0 for coarse column j1, then axis 1
            auto t0 = [&](int j1) { return tail_interp<T>(i0, m, [&](int j0) { return e[tidx(Lc, j0, j1, 0)]; }); };
            val = tail_interp<T>(i1, m, t0);
        } else {
            const int i0 = tdiv(q, n * n), rem = q - i0 * n * n, i1 = tdiv(rem, n), i2 = rem - i1 * n;
            p = tidx(Lf, i0, i1, i2);
            auto t1 = [&](int j2) {
                auto t0 = [&](int j1) {
                    return tail_interp<T>(i0, m, [&](int j0) { return e[tidx(Lc, j0, j1, j2)]; });
                };
                return tail_interp<T>(i1, m, t0);
            };
            val = tail_interp<T>(i2, m, t1);
        }
        xo[p] = O::add(xi[p], val);
    }
}

// barrier `id` over the first n threads (n a multiple of 32): the small levels of the tail only
// occupy a few warps, and only those wait for each other.  Warps that skip small ops run ahead
// to the next barrier that includes them, so every distinct count has its own barrier id (the
// host assigns them; id 0 = all threads = __syncthreads).
__device__ __forceinline__ void tbar(int id, int n) {
    if (id == 0) {
        __syncthreads();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    }
}

// getrs order (Appendix A.5/A.6), identical to k_coarse_solve, in one warp (nlu <= 32): lane i
// holds y_i; the row interchanges, the column-oriented FMA forward substitution and the
// true-divide back substitution run in the sequential j order through shuffles
template <class T>
__device__ void tail_coarse_warp(const TailLevel<T>& v, const T* lu, const int* piv, int nlu) {
    using O = Op<T>;
    const Layout& L = v.L;
    const int l = threadIdx.x;
    T y = l < nlu ? v.b[tpoint(L, l)] : T(0);
    for (int i = 0; i < nlu; ++i) {
        const int p = piv[i];
        if (p != i) {
            const T yi = __shfl_sync(0xffffffffu, y, i), yp = __shfl_sync(0xffffffffu, y, p);
            if (l == i) y = yp;
            if (l == p) y = yi;
        }
    }
    for (int j = 0; j < nlu; ++j) {
        const T yj = __shfl_sync(0xffffffffu, y, j);
        if (l > j && l < nlu) y = O::fma(-lu[(long long)l * nlu + j], yj, y);
    }
    for (int j = nlu - 1; j >= 0; --j) {
        if (l == j) y = O::div(y, lu[(long long)j * nlu + j]);
        const T yj = __shfl_sync(0xffffffffu, y, j);
        if (l < j) y = O::fma(-lu[(long long)l * nlu + j], yj, y);
    }
    if (l < nlu) v.x[0][tpoint(L, l)] = y;
}

// getrs order (Appendix A.5/A.6), identical to k_coarse_solve, over the first n threads
template <class T>
__device__ void tail_coarse_phase(const TailLevel<T>& v, T* y, const T* lu, const int* piv, int nlu, int id, int n) {
    using O = Op<T>;
    const Layout& L = v.L;
    for (int q = threadIdx.x; q < nlu; q += blockDim.x) y[q] = v.b[tpoint(L, q)];
    tbar(id, n);
    if (threadIdx.x == 0) {
        for (int i = 0; i < nlu; ++i) {
            const int p = piv[i];
            if (p != i) {
                const T t = y[i];
                y[i] = y[p];
                y[p] = t;
            }
        }
    }
    tbar(id, n);
    for (int j = 0; j < nlu; ++j) {
        const T yj = y[j];
        for (int i = j + 1 + threadIdx.x; i < nlu; i += n) y[i] = O::fma(-lu[(long long)i * nlu + j], yj, y[i]);
        tbar(id, n);
    }
    for (int j = nlu - 1; j >= 0; --j) {
        if (threadIdx.x == 0) y[j] = O::div(y[j], lu[(long long)j * nlu + j]);
        tbar(id, n);
        const T yj = y[j];
        for (int i = threadIdx.x; i < j; i += n) y[i] = O::fma(-lu[(long long)i * nlu + j], yj, y[i]);
        tbar(id, n);
    }
    for (int q = threadIdx.x; q < nlu; q += blockDim.x) v.x[0][tpoint(L, q)] = y[q];
}

// copy the interior of one level between two layouts (global padded <-> shared compact)
template <class T, bool SRC_GLOBAL>
__device__ void tail_copy(const Layout& Ld, T* dst, const Layout& Ls, const T* src) {
    const int cnt = npoints(Ld);
    for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
        // global sources through L2: in the cluster tail other CTAs of the cluster wrote them
        if constexpr (SRC_GLOBAL) {
            dst[tpoint(Ld, q)] = __ldcg(src + tpoint(Ls, q));
        } else {
            dst[tpoint(Ld, q)] = src[tpoint(Ls, q)];
        }
    }
}

template <class T, int S>
__device__ void tail_body(const TailArgs<T>& a, unsigned char* smem_raw) {
    // [level descriptors | ops | level arrays | LU work vector y]
    TailLevel<T>* lv = reinterpret_cast<TailLevel<T>*>(smem_raw);
    TailOp* ops = reinterpret_cast<TailOp*>(lv + a.nlv);
    T* arr = reinterpret_cast<T*>(smem_raw + a.arr_off);
    T* y = arr + a.arr_elems;
    for (int i = threadIdx.x; i < a.nlv; i += blockDim.x) {
        TailLevel<T> v = a.lv[i];  // host-built: the array "pointers" are element offsets into arr
        for (int k = 0; k < 2; ++k) v.x[k] = arr + reinterpret_cast<size_t>(v.x[k]);
        v.b = arr + reinterpret_cast<size_t>(v.b);
        v.r = arr + reinterpret_cast<size_t>(v.r);
        lv[i] = v;
    }
    for (int i = threadIdx.x; i < a.nops; i += blockDim.x) ops[i] = a.ops[i];
    for (int i = threadIdx.x; i < a.arr_elems; i += blockDim.x) arr[i] = T(0);
    __syncthreads();
    // entry level: b (and the start iterate) from its global buffers
    tail_copy<T, true>(lv[0].L, lv[0].b, a.gL, a.gb);
    if (!a.entry_fz) tail_copy<T, true>(lv[0].L, lv[0].x[a.entry_a], a.gL, a.gx_in);
    __syncthreads();
    for (int i = 0; i < a.nops; ++i) {
        const TailOp op = ops[i];
        // the threads of op i and of op i-1 (always a prefix of warps) meet here
        if ((int)threadIdx.x >= op.npre) continue;
        if (i > 0) tbar(op.bid_pre, op.npre);
        if ((int)threadIdx.x >= op.nthr) continue;
        const TailLevel<T>& v = lv[op.level];
        switch (op.type) {
            case TAIL_SWEEP:
                tail_residual_phase<T>(v, v.x[op.a_in], op.fz);
                tbar(op.bid_in, op.nthr);
                tail_relax_phase<T, S>(v, op.fz ? nullptr : v.x[op.a_in], v.x[op.a_out], a.M, a.omega);
                break;
            case TAIL_ZERO: {
                const int cnt = npoints(v.L);
                for (int q = threadIdx.x; q < cnt; q += blockDim.x) v.x[op.a_out][tpoint(v.L, q)] = T(0);
                break;
            }
            case TAIL_RESTRICT:
                tail_residual_phase<T>(v, v.x[op.a_in], false);
                tbar(op.bid_in, op.nthr);
                tail_restrict_phase<T>(v, lv[op.level + 1]);
                break;
            case TAIL_PROLONG: {
                const TailLevel<T>& c = lv[op.level + 1];
                tail_prolong_phase<T>(v, c, v.x[op.a_in], v.x[op.a_out], c.x[op.c]);
                break;
            }
            case TAIL_COARSE:
                if (a.nlu <= 32)
                    tail_coarse_warp<T>(v, a.lu, a.piv, a.nlu);
                else
                    tail_coarse_phase<T>(v, y, a.lu, a.piv, a.nlu, op.bid_in, op.nthr);
                break;
        }
    }
    __syncthreads();
    tail_copy<T, false>(a.gL, a.gx_out, lv[0].L, lv[0].x[a.out_a]);
}

template <class T, int S>
__global__ void __launch_bounds__(kTailThreads) k_tail(TailArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    tail_body<T, S>(a, smem_raw);
}

// ------------------------------------------------------------------------------------------
// Cluster tail: the middle levels (above the shared-memory tail) run on a 16-CTA thread-block
// cluster over their global (L2-resident) level buffers, point-parallel, phases separated by
// hardware cluster barriers (barrier.cluster arrive.release / wait.acquire, ~0.7 us with an L2
// round trip against several us per dependent kernel); the smallest levels then run as the
// shared-memory tail in CTA 0 (TAIL_SOLO) while the other CTAs wait at the next barrier.
// Cross-CTA data is read with ld.global.cg (L2).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ unsigned cluster_rank() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ unsigned cluster_size() {
    unsigned r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}

template <class T>
__device__ __forceinline__ T cg_residual(const Layout& L, const T* x, const T* b, long long p, T sA) {
    if (L.dim == 2)
        return residual2d<T>(__ldcg(b + p), __ldcg(x + p), __ldcg(x + p + L.px), __ldcg(x + p - L.px), __ldcg(x + p + 1),
                             __ldcg(x + p - 1), sA);
    return residual3d<T>(__ldcg(b + p), __ldcg(x + p), __ldcg(x + p + L.pp), __ldcg(x + p - L.pp), __ldcg(x + p + L.px),
                         __ldcg(x + p - L.px), __ldcg(x + p + 1), __ldcg(x + p - 1), sA);
}

template <class T>
__device__ void cl_op(const ClusterArgs<T>& a, const TailOp& op, int start, int stride) {
    using O = Op<T>;
    const TailLevel<T>& v = a.lv[op.level];
    const Layout& L = v.L;
    const int cnt = npoints(L);
    switch (op.type) {
        case TAIL_SWEEP: {
            for (int q = start; q < cnt; q += stride) {
                const long long p = gpoint(L, q);
                v.r[p] = op.fz ? __ldcg(v.b + p) : cg_residual<T>(L, v.x[op.a_in], v.b, p, v.sA);
            }
            cluster_sync_all();
            const T* x = op.fz ? nullptr : v.x[op.a_in];
            T* xo = v.x[op.a_out];
            for (int q = start; q < cnt; q += stride) {
                const long long p = gpoint(L, q);
                T acc = T(0);
                for (int k = 0; k < a.M.nt; ++k) {
                    const long long o = L.dim == 2 ? (long long)a.M.off[k][0] * L.px + a.M.off[k][1]
                                                   : (long long)a.M.off[k][0] * L.pp + (long long)a.M.off[k][1] * L.px +
                                                         a.M.off[k][2];
                    acc = O::add(acc, O::mul(a.M.c[k], __ldcg(v.r + p + o)));
                }
                xo[p] = relax<T>(x ? __ldcg(x + p) : T(0), acc, v.sM, a.omega);
            }
            break;
        }
        case TAIL_ZERO:
            for (int q = start; q < cnt; q += stride) v.x[op.a_out][gpoint(L, q)] = T(0);
            break;
        case TAIL_RESTRICT: {
            for (int q = start; q < cnt; q += stride) {
                const long long p = gpoint(L, q);
                v.r[p] = cg_residual<T>(L, v.x[op.a_in], v.b, p, v.sA);
            }
            cluster_sync_all();
            const TailLevel<T>& c = a.lv[op.level + 1];
            const Layout& Lc = c.L;
            const int m = Lc.n;
            const int cc = npoints(Lc);
            const T* r = v.r;
            for (int q = start; q < cc; q += stride) {
                if (L.dim == 2) {
                    const int I = tdiv(q, m), K = q - I * m;
                    T t[3];
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        const long long p = gidx(L, 2 * I + 1, 2 * K + k, 0);
                        t[k] = fw<T>(__ldcg(r + p - L.px), __ldcg(r + p), __ldcg(r + p + L.px));
                    }
                    c.b[gidx(Lc, I, K, 0)] = fw<T>(t[0], t[1], t[2]);
                } else {
                    const int I = tdiv(q, m * m), rem = q - I * m * m, J = tdiv(rem, m), K = rem - J * m;
                    T u[3];
#pragma unroll
                    for (int qk = 0; qk < 3; ++qk) {
                        T t[3];
#pragma unroll
                        for (int qj = 0; qj < 3; ++qj) {
                            const long long p = gidx(L, 2 * I + 1, 2 * J + qj, 2 * K + qk);
                            t[qj] = fw<T>(__ldcg(r + p - L.pp), __ldcg(r + p), __ldcg(r + p + L.pp));
                        }
                        u[qk] = fw<T>(t[0], t[1], t[2]);
                    }
                    c.b[gidx(Lc, I, J, K)] = fw<T>(u[0], u[1], u[2]);
                }
            }
            break;
        }
        case TAIL_PROLONG: {
            const TailLevel<T>& c = a.lv[op.level + 1];
            const Layout& Lc = c.L;
            const int m = Lc.n, n = L.n;
            const T* e = c.x[op.c];
            const T* xi = v.x[op.a_in];
            T* xo = v.x[op.a_out];
            for (int q = start; q < cnt; q += stride) {
                T val;
                long long p;
                if (L.dim == 2) {
                    const int i0 = q / n, i1 = q % n;
                    p = gidx(L, i0, i1, 0);
                    auto t0 = [&](int j1) {
                        return tail_interp<T>(i0, m, [&](int j0) { return __ldcg(e + gidx(Lc, j0, j1, 0)); });
                    };
                    val = tail_interp<T>(i1, m, t0);
                } else {
                    const int i0 = tdiv(q, n * n), rem = q - i0 * n * n, i1 = tdiv(rem, n), i2 = rem - i1 * n;
                    p = gidx(L, i0, i1, i2);
                    auto t1 = [&](int j2) {
                        auto t0 = [&](int j1) {
                            return tail_interp<T>(i0, m, [&](int j0) { return __ldcg(e + gidx(Lc, j0, j1, j2)); });
                        };
                        return tail_interp<T>(i1, m, t0);
                    };
                    val = tail_interp<T>(i2, m, t1);
                }
                xo[p] = O::add(__ldcg(xi + p), val);
            }
            break;
        }
        default:
            break;
    }
}

template <class T>
__global__ void __launch_bounds__(kTailThreads) k_cluster_tail(ClusterArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    const unsigned rank = cluster_rank();
    const int start = (int)(rank * blockDim.x + threadIdx.x), stride = (int)(cluster_size() * blockDim.x);
    for (int i = 0; i < a.nops; ++i) {
        const TailOp op = a.ops[i];
        if (i > 0) cluster_sync_all();
        if (op.type == TAIL_SOLO) {
            if (rank == 0) tail_body<T, SHAPE_GENERIC>(a.solo[op.a_in][op.fz], smem_raw);
        } else {
            cl_op<T>(a, op, start, stride);
        }
    }
}

template <class T>
cudaError_t cluster_occupancy(int csize, size_t smem, int* nclusters) {
    cudaError_t e = cudaFuncSetAttribute(k_cluster_tail<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(k_cluster_tail<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kTailThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaOccupancyMaxActiveClusters(nclusters, k_cluster_tail<T>, &cfg);
}

template <class T>
cudaError_t launch_cluster_tail(const ClusterArgs<T>& a, int csize, size_t smem, cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(k_cluster_tail<T>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
    if (smem > 48 * 1024) {
        e = cudaFuncSetAttribute(k_cluster_tail<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(csize);
    cfg.blockDim = dim3(kTailThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = csize;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k_cluster_tail<T>, a);
}

template <class T, int S>
static cudaError_t launch_tail_s(const TailArgs<T>& a, cudaStream_t s) {
    if (a.smem > 48 * 1024) {  // per device, so set on every launch (host-side, cheap)
        cudaError_t e = cudaFuncSetAttribute(k_tail<T, S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem);
        if (e != cudaSuccess) return e;
    }
    return launch_pdl(k_tail<T, S>, dim3(1), dim3(kTailThreads), a.smem, s, a);
}

template <class T>
cudaError_t launch_tail(const TailArgs<T>& a, cudaStream_t s) {
    const int dim = a.gL.dim;
    switch (a.shape) {
        case SHAPE_C1: return launch_tail_s<T, SHAPE_C1>(a, s);
        case SHAPE_STAR5:
            if (dim == 2) return launch_tail_s<T, SHAPE_STAR5>(a, s);
            break;
        case SHAPE_BOX9:
            if (dim == 2) return launch_tail_s<T, SHAPE_BOX9>(a, s);
            break;
        case SHAPE_STAR7:
            if (dim == 3) return launch_tail_s<T, SHAPE_STAR7>(a, s);
            break;
        default: break;
    }
    return launch_tail_s<T, SHAPE_GENERIC>(a, s);
}

template cudaError_t launch_tail<double>(const TailArgs<double>&, cudaStream_t);
template cudaError_t launch_tail<float>(const TailArgs<float>&, cudaStream_t);
template cudaError_t launch_cluster_tail<double>(const ClusterArgs<double>&, int, size_t, cudaStream_t);
template cudaError_t cluster_occupancy<double>(int, size_t, int*);
template cudaError_t cluster_occupancy<float>(int, size_t, int*);
template cudaError_t launch_cluster_tail<float>(const ClusterArgs<float>&, int, size_t, cudaStream_t);

}  // namespace spaimg
