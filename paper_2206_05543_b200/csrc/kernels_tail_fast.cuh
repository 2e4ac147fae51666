// K5+ fast path: the shared-memory coarse engine with the V/W recursion compiled in, for
// power-of-two hierarchies (every level has n = 2^k - 1 interior points per axis, frame 1) --
// every BASELINE configuration.  The level geometry, each op's warp count and the barrier before
// it are compile-time constants, so an op is straight-line code: barrier, shared-memory tile
// loads, the Appendix-A arithmetic, stores.  The generic interpreter (kernels_tail.cu) pays two
// to three dependent indexed constant/shared-memory lookups and jump-table branches per op
// (~200-500 cycles, measured with SPAIMG_TAIL_PROF=1) on top of a ~110-cycle op
// (tools/op_probe.cu).
//
// Barriers: every point op on level l runs on P(l) warps (its W^dim box over 512 threads), the
// restriction onto level l+1 on P(l+1) warps, the coarse solve on one.  The barrier before an op
// spans the warps of the op and of its predecessor, which is statically known: within a visit
// of level l every predecessor is an op on level l (or the restriction, P(l+1) <= P(l)); the
// first op of a visit of level l+1 follows either the restriction (P(l+1) warps) or the
// previous visit of l+1 (whose last op runs on P(l+1) warps); the prolongation of level l
// follows the last op of a visit of l+1.  One named barrier id per warp count.
#pragma once

#include <climits>

#include "tail_ops.cuh"

namespace spaimg {

template <int BW>
__device__ __forceinline__ void fast_sync() {
    if constexpr (BW >= NT / 32) {
        __syncthreads();
    } else if constexpr (BW == 1) {
        __syncwarp();
    } else {
        constexpr int ID = BW == 2 ? 1 : BW == 4 ? 2 : BW == 8 ? 3 : 4;
        asm volatile("bar.sync %0, %1;" ::"n"(ID), "n"(BW * 32) : "memory");
    }
}

template <class T, int S, int D, int LE, int LC>
struct FastTail {
    static constexpr int NL = LE - LC + 1;  // shared-memory levels, the last one the coarse level
    __host__ __device__ static constexpr int logw(int l) { return LE - l; }
    __host__ __device__ static constexpr int n(int l) { return (1 << (LE - l)) - 1; }
    __host__ __device__ static constexpr int w(int l) { return n(l) + 2; }
    __host__ __device__ static constexpr int s0(int l) { return D == 2 ? w(l) : w(l) * w(l); }
    __host__ __device__ static constexpr int s1(int l) { return D == 3 ? w(l) : 0; }
    __host__ __device__ static constexpr int size(int l) {
        return ((D == 2 ? w(l) * w(l) : w(l) * w(l) * w(l)) + 1) / 2 * 2;
    }
    __host__ __device__ static constexpr int origin(int l) { return s0(l) + s1(l) + 1; }
    __host__ __device__ static constexpr int narr(int l) { return l == NL - 1 ? 2 : 3; }
    __host__ __device__ static constexpr int base(int l) {
        int c = 0;
        for (int k = 0; k < l; ++k) c += narr(k) * size(k);
        return c;
    }
    __device__ static int base_rt(int l) { return base(l); }
    __device__ static int size_rt(int l) { return size(l); }
    __host__ __device__ static constexpr int xo(int l) { return base(l) + origin(l); }
    __host__ __device__ static constexpr int bo(int l) { return base(l) + size(l) + origin(l); }
    __host__ __device__ static constexpr int ro(int l) { return base(l) + 2 * size(l) + origin(l); }
    // the array block (+ two axis-0 rows of slack for the strips' unused over-reads), then the
    // coarse factors (T) and their gather / scatter offsets (int)
    __host__ __device__ static constexpr int elems() { return base(NL) + 2 * s0(0) + 2 * s1(0) + 2; }
    __host__ __device__ static constexpr int cf_off() { return elems(); }
    __host__ __device__ static constexpr int cf_elems() { return (NLU * NLU + 2 * NLU + 1) / 2 * 2; }
    __host__ __device__ static constexpr size_t smem_bytes() {
        return (size_t)(elems() + cf_elems()) * sizeof(T) + 2 * NLU * sizeof(int);
    }
    __host__ __device__ static constexpr int zero_from() { return base(0) + 2 * size(0); }
    // threads of a level's point ops.  (Measured and rejected: running the small levels in ONE
    // warp with K-point strips and __syncwarp between ops -- a lone warp is issue-bound on one
    // SMSP, and the W(1,0) engine entry got 14 % slower than with the ops spread over the CTA.)
    __host__ __device__ static constexpr int NTH(int) { return NT; }
    __host__ __device__ static constexpr int warps(int lw, int nth) {
        const int pts = 1 << (D * lw);
        const int act = pts >= nth ? nth : pts;
        return act >= 32 ? act / 32 : 1;
    }
    __host__ __device__ static constexpr int P(int l) { return warps(logw(l), NTH(l)); }
    // the restriction of level l onto l+1 is mapped like a point op of level l+1
    __host__ __device__ static constexpr int PF(int l) { return warps(logw(l) - 1, NTH(l + 1)); }
    static constexpr int NLU = D == 2 ? (LC == 1 ? 1 : 9) : (LC == 1 ? 1 : 27);

    // the level geometry as the op bodies take it (compile-time fields fold into the addresses)
    __device__ static __forceinline__ TailLv<T> geo(const TailArgs<T>& a, int l) {
        TailLv<T> g;
        g.n = n(l);
        g.logw = logw(l);
        g.s0 = s0(l);
        g.s1 = s1(l);
        g.x = xo(l);
        g.b = bo(l);
        g.r = ro(l);
        g.pad = 0;
        g.sA = a.lv[l].sA;
        g.sM = a.lv[l].sM;
        return g;
    }

    // one op: barrier over BW warps, then the op on NW warps (pc: op counter for SPAIMG_TAIL_PROF)
    template <int BW, int NW, class Fn>
    __device__ static __forceinline__ void step(const TailArgs<T>& a, int warp, int& pc, Fn&& fn) {
        if (warp < BW) {
            fast_sync<BW>();
            SPAIMG_JITTER();
            if (a.prof && threadIdx.x == 0) a.prof[pc] = clock64();
            if (warp < NW) fn();
        }
        ++pc;
    }

    // residual + restriction in one op (tail_ops.cuh op_resfw) where the coarse box maps one point
    // per thread, 2D only.  Measured per op with SPAIMG_TAIL_PROF and per cycle with
    // tools/tail_variants.sh: in 3D the 27-point footprint costs more than the barrier it saves
    // (n = 7: 1656 cycles fused, ~850 as residual, barrier, restriction; c3 V(1,1) 117 -> 114
    // us/cycle unfused); in 2D it is neutral.  A fused prolongation + next residual (every thread
    // interpolating the correction at its point and its 2 D neighbours) was removed: it cost 1100
    // cycles against ~730 unfused at n = 15 in 2D and 6600 against ~2100 at n = 7 in 3D; without
    // it c2 W(1,0) went 2.46 -> 2.28 ms/cycle, c2 V(1,1) 0.379 -> 0.373, c3 V(1,1) 127 -> 117 us.
    __host__ __device__ static constexpr bool fuse_rr(int l) {
        return D == 2 && l + 1 < NL && (1 << (D * (LE - l - 1))) <= NTH(l + 1);
    }

    // visit of level L (multigrid.py:157-185); fz: from a zero iterate
    template <int L>
    __device__ static __forceinline__ void visit(const TailArgs<T>& a, T* arr, int warp, int& pc, bool fz) {
        constexpr int PL = P(L), PC = PF(L), LW = logw(L), TL = NTH(L), TC = NTH(L + 1);
        const TailLv<T> f = geo(a, L);
        const TailLv<T> c = geo(a, L + 1);
        for (int k = 0; k < a.nu1; ++k) {
            if (fz && k == 0) {
                step<PL, PL>(a, warp, pc, [&] { op_relax<T, S, D, LW, true, TL>(f, arr, a.M, a.omega); });
            } else {
                step<PL, PL>(a, warp, pc, [&] { op_res<T, D, LW, TL>(f, arr); });
                step<PL, PL>(a, warp, pc, [&] { op_relax<T, S, D, LW, false, TL>(f, arr, a.M, a.omega); });
            }
        }
        if (fz && a.nu1 == 0) step<PL, PL>(a, warp, pc, [&] { op_zero<T, D, LW, TL>(f, arr); });
        if constexpr (fuse_rr(L)) {
            step<PL, PC>(a, warp, pc, [&] { op_resfw<T, D, LW, TC>(f, c, arr); });
        } else {
            step<PL, PL>(a, warp, pc, [&] { op_res<T, D, LW, TL>(f, arr); });
            step<PL, PC>(a, warp, pc, [&] { op_fw<T, D, LW, TC>(f, c, arr); });
        }
        if constexpr (L + 1 == NL - 1) {
            // direct solve (multigrid.py:178-179): once, whatever gamma (the reference solves the
            // restricted system directly instead of cycling on it)
            const T* cf = arr + cf_off();
            const int* ci = reinterpret_cast<const int*>(cf + cf_elems());
            step<PC, 1>(a, warp, pc, [&] {
                if (threadIdx.x == 0) coarse_fast<T, NLU>(cf, ci, arr + bo(L + 1), arr + xo(L + 1));
            });
        } else {
            for (int g = 0; g < a.gamma; ++g) visit<L + 1>(a, arr, warp, pc, g == 0);
        }
        // prolongation + correction (multigrid.py:184)
#ifdef SPAIMG_DEBUG_BREAK_BARRIER
        // fault injection for the checked-build self-test (tools/README): no barrier before the
        // prolongation, so it may read the coarse correction before the coarse visit wrote it
        if (warp < PL) op_prolong<T, D, LW, TL>(f, c, arr);
        ++pc;
#else
        step<PL, PL>(a, warp, pc, [&] { op_prolong<T, D, LW, TL>(f, c, arr); });
#endif
        for (int k = 0; k < a.nu2; ++k) {
            step<PL, PL>(a, warp, pc, [&] { op_res<T, D, LW, TL>(f, arr); });
            step<PL, PL>(a, warp, pc, [&] { op_relax<T, S, D, LW, false, TL>(f, arr, a.M, a.omega); });
        }
    }

    // entry level in: b (and the start iterate unless the entry is from zero) of the box
    // [-1, n+1)^D of the global padded layout, whose frame is zero.  Compile-time geometry: the
    // loop is fully unrolled and every global load is issued before the first store (a rolled
    // loop waited out one L2 round trip per iteration).
    __device__ static __forceinline__ void load_entry(const TailArgs<T>& a, T* arr, bool fz) {
        constexpr int W0 = w(0), CNT = D == 2 ? W0 * W0 : W0 * W0 * W0;
        constexpr int IT = (CNT + NT - 1) / NT, UB = IT;  // one batch: every load in flight at once
        const long long p0 = D == 2 ? a.gL.px : a.gL.pp;
#pragma unroll 1
        for (int ib = 0; ib < IT; ib += UB) {
            T vb[UB], vx[UB];
            int so[UB];
#pragma unroll
            for (int u = 0; u < UB; ++u) {
                const int qq = (ib + u) * NT + (int)threadIdx.x;
                so[u] = INT_MIN;
                vb[u] = vx[u] = T(0);
                if (ib + u < IT && qq < CNT) {
                    const int j0 = (D == 2 ? qq / W0 : qq / (W0 * W0)) - 1;
                    const int rem = D == 2 ? 0 : qq % (W0 * W0);
                    const int j1 = D == 2 ? 0 : rem / W0 - 1;
                    const int j2 = (D == 2 ? qq % W0 : rem % W0) - 1;
                    const long long g = a.gL.origin + (long long)j0 * p0 + (D == 3 ? (long long)j1 * a.gL.px : 0LL) + j2;
                    so[u] = j0 * s0(0) + j1 * s1(0) + j2;
                    vb[u] = a.gb[g];
                    if (!fz) vx[u] = a.gx[g];
                }
            }
#pragma unroll
            for (int u = 0; u < UB; ++u)
                if (so[u] != INT_MIN) {
                    arr[bo(0) + so[u]] = vb[u];
                    arr[xo(0) + so[u]] = vx[u];
                }
        }
    }

    // entry level out: the iterate's interior back to the global padded layout
    __device__ static __forceinline__ void store_entry(const TailArgs<T>& a, const T* arr) {
        constexpr int N0 = n(0), CNT = D == 2 ? N0 * N0 : N0 * N0 * N0;
        const long long p0 = D == 2 ? a.gL.px : a.gL.pp;
#pragma unroll 4
        for (int qq = threadIdx.x; qq < CNT; qq += NT) {
            const int j0 = D == 2 ? qq / N0 : qq / (N0 * N0);
            const int rem = D == 2 ? 0 : qq % (N0 * N0);
            const int j1 = D == 2 ? 0 : rem / N0;
            const int j2 = D == 2 ? qq % N0 : rem % N0;
            a.gx[a.gL.origin + (long long)j0 * p0 + (D == 3 ? (long long)j1 * a.gL.px : 0LL) + j2] =
                arr[xo(0) + j0 * s0(0) + j1 * s1(0) + j2];
        }
    }

    __device__ static __forceinline__ void run(const TailArgs<T>& a, T* arr) {
        const int t = threadIdx.x;
        if (a.prof && t == 0) a.prof[2 * kTailMaxOps] = clock64();  // kernel entry (SPAIMG_TAIL_PROF)
        load_entry(a, arr, a.entry_fz != 0);
        for (int i = zero_from() + t; i < elems(); i += NT) arr[i] = T(0);
        if constexpr (kDebugChecks) {
            __syncthreads();
#pragma unroll 1
            for (int l = 0; l < NL; ++l) {
                const int nn = (1 << (LE - l)) - 1, w0 = nn + 2;
                const int t0 = D == 2 ? w0 : w0 * w0, t1 = D == 3 ? w0 : 0;
                const int bl = base_rt(l), sz = size_rt(l), org = t0 + t1 + 1;
                if (l > 0) {
                    tail_poison<T, D>(arr, nn, 1, t0, t1, bl + org);
                    tail_poison<T, D>(arr, nn, 1, t0, t1, bl + sz + org);
                }
                if (l < NL - 1) tail_poison<T, D>(arr, nn, 1, t0, t1, bl + 2 * sz + org);
            }
            for (int i = base(NL) + t; i < elems(); i += NT) arr[i] = T(__int_as_float(0x7fc00000));
        }
        T* cf = arr + cf_off();
        int* ci = reinterpret_cast<int*>(cf + cf_elems());
        for (int i = t; i < NLU * NLU; i += NT) cf[i] = a.lu[i];
        if (t < NLU) {
            cf[NLU * NLU + t] = a.dg[t];
            cf[NLU * NLU + NLU + t] = a.rc[t];
            ci[t] = a.cin[t];
            ci[NLU + t] = a.cout[t];
        }
        __syncthreads();
        int pc = 0;
        visit<0>(a, arr, t >> 5, pc, a.entry_fz != 0);
        __syncthreads();
        if (a.prof && t == 0) a.prof[pc] = clock64();
        store_entry(a, arr);
        if (a.prof) {
            __syncthreads();
            if (t == 0) a.prof[2 * kTailMaxOps + 1] = clock64();  // kernel exit
        }
    }
};

template <class T, int S, int D, int LE, int LC>
__global__ void __launch_bounds__(NT, 1) k_tail_fast(const __grid_constant__ TailArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    FastTail<T, S, D, LE, LC>::run(a, reinterpret_cast<T*>(smem));
}

template <class T, int S, int D, int LE, int LC>
static cudaError_t launch_tail_fast_s(const TailArgs<T>& a, cudaStream_t s) {
    constexpr size_t smem = FastTail<T, S, D, LE, LC>::smem_bytes();
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_tail_fast<T, S, D, LE, LC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    return launch_k(k_tail_fast<T, S, D, LE, LC>, dim3(1), dim3(NT), smem, s, a);
}

}  // namespace spaimg
