// K1 + K2 fused on the 2D marching levels: the last pre-smoothing sweep x' = x + omega M (b - A x)
// (reference multigrid.py:98-100) and the residual + full-weighting restriction of its result
// bc = restrict(b - A x') (multigrid.py:176-177, :104-119) in ONE row march, so neither x' nor b
// is read back from HBM for the restriction: x + b in, x' + bc out (26 B per unknown in fp64
// instead of 24 + 18).  Optionally the norm of the input residual rides along (part A of the
// solve loop, as in the plain sweep).
//
// A CTA owns a strip of W fine columns (W/2 coarse columns) and a chunk of rows (even, so that
// coarse rows partition across chunks) and marches down the rows.  Per step j:
//   before the barrier: r(j) on the strip (consumers, registers) and at 5 halo columns (producer
//                       lanes), into a 4-row shared r ring; b(j) into a 5-row shared b ring;
//   after the barrier:  x'(j-1) from r(j-2..j) (consumers: own columns, to HBM and a 4-row shared
//                       x' ring; producer lanes: x' at c0-1, c0+W, c0+W+1);
//                       r'(j-3) = b - A x' from the x' ring (consumers own columns; one producer
//                       lane at column c0+W for the strip-edge weight);
//                       the full weighting of coarse row (j-6)/2 from the axis-0 weights formed
//                       one step earlier (warp-edge and strip-edge weights through shared slots).
// Every value crosses at least one barrier between its producer and its consumers, and every
// expression is the reference's tree (spaimg_common.cuh), so the result is bitwise that of the
// separate sweep and K2 kernels.
#include <cstdlib>

#include "kernels.h"
#include "march.cuh"
#include "ptx.cuh"

namespace spaimg {

constexpr int PR_NW = 4;  // consumer warps
constexpr int PR_ST = 6;  // (x, b) stage ring depth (= step unroll)
constexpr int PR_H = 4;   // staged halo columns on each side

template <class T> struct PRG {
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int W = 32 * VEC * PR_NW;
    static constexpr int RW = W + 2 * PR_H;
    static constexpr size_t smem = (size_t)(2 * PR_ST + 4 + 4 + 5) * RW * sizeof(T) + (PR_NW + 1) * 2 * sizeof(T) +
                                   PR_ST * 8 + 16;
};

template <class T>
struct PRCtx {
    T* xs;  // x stages
    T* bs;  // b stages
    T* rr;  // r ring (4 rows)
    T* xp;  // x' ring (4 rows)
    T* bp;  // b ring (5 rows)
    T* te;  // edge axis-0 weights: te[w] = first weight of consumer warp w, te[NW] = strip edge
    uint64_t* full;
    const T* xrow0;
    const T* brow0;
    T* orow0;   // x' row 0, own first column
    T* crow0;   // coarse row 0 at the lane's first coarse column
    long long px, cpx;
    int n, m, c0, col, sidx, q0, q_last, r0, r_end, I0, I1, lane, warp;
    bool producer, last_strip;
};

template <class T>
__device__ __forceinline__ T* pr_row(T* ring, int nrows, int row) {
    constexpr int RW = PRG<T>::RW;
    return ring + ((row % nrows + nrows) % nrows) * RW;
}

template <class T, bool FZ>
__device__ __forceinline__ void pr_issue(const PRCtx<T>& c, int q, int slot) {
    constexpr int RW = PRG<T>::RW;
    constexpr uint32_t row_bytes = RW * sizeof(T);
    // rows past the ghost frame are never used (masked); stage a zero frame row instead
    const int src = q < -2 ? -2 : (q > c.n + 1 ? c.n + 1 : q);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&c.full[slot], FZ ? row_bytes : 2 * row_bytes);
    if (!FZ) bulk_g2s(c.xs + slot * RW, c.xrow0 + (long long)src * c.px, row_bytes, &c.full[slot]);
    bulk_g2s(c.bs + slot * RW, c.brow0 + (long long)src * c.px, row_bytes, &c.full[slot]);
}

template <class T, int S, bool FZ, bool NORM, int P>
__device__ __forceinline__ void pr_step(const PRCtx<T>& c, int k, T (&X)[3][PRG<T>::VEC], T (&R)[3][PRG<T>::VEC],
                                        T (&RL)[3], T (&RH)[3], T (&RP)[3][PRG<T>::VEC], T (&TP)[PRG<T>::VEC],
                                        T (&RE)[3], const Terms<T>& M, T sA, T sM, T omega, double& nacc) {
    using O = Op<T>;
    using G = PRG<T>;
    constexpr int VEC = G::VEC;
    constexpr int W = G::W;
    constexpr int RW = G::RW;
    constexpr int ST = PR_ST;
    constexpr int H = PR_H;
    constexpr int sj = P % ST, sp = (P + 1) % ST, sm = (P + ST - 1) % ST;  // stage slots of rows j, j+1, j-1
    constexpr int ic = P % 3, ip = (P + 1) % 3, im = (P + 2) % 3;          // register rows j, j+1 (X) / j-2 (R), j-1
    const int j = c.q0 + k;
    mbar_wait(&c.full[sp], (uint32_t)(((k + 1) / ST) & 1));
    const bool row_in = (unsigned)j < (unsigned)c.n;
    T* rrow = pr_row(c.rr, 4, j);
    // ---------------- before the barrier: r(j) --------------------------------------------
    if (!c.producer) {
        T bj[VEC];
        V16<T>::ld(c.bs + sj * RW + c.sidx, bj);
        V16<T>::st(pr_row(c.bp, 5, j) + c.sidx, bj);
        if constexpr (FZ) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) R[ic][v] = bj[v];
        } else {
            V16<T>::ld(c.xs + sp * RW + c.sidx, X[ip]);
            const T left = c.xs[sj * RW + c.sidx - 1];
            const T right = c.xs[sj * RW + c.sidx + VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                const T xe = v + 1 < VEC ? X[ic][v + 1] : right;
                const T xw = v > 0 ? X[ic][v - 1] : left;
                R[ic][v] = residual2d<T>(bj[v], X[ic][v], X[ip][v], X[im][v], xe, xw, sA);
            }
        }
        if (!row_in || c.last_strip) {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (!row_in || c.col + v >= c.n) R[ic][v] = T(0);
        }
        if (NORM && j >= c.r0 && j < c.r_end) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) nacc += (double)R[ic][v] * (double)R[ic][v];
        }
        V16<T>::st(rrow + c.sidx, R[ic]);
    } else if (c.lane < 5) {
        // halo residuals at c0-2, c0-1, c0+W, c0+W+1, c0+W+2
        const int off = c.lane < 2 ? c.lane - 2 : W + c.lane - 2;
        const int si = H + off, cc = c.c0 + off;
        T rv;
        if constexpr (FZ) {
            rv = c.bs[sj * RW + si];
        } else {
            rv = residual2d<T>(c.bs[sj * RW + si], c.xs[sj * RW + si], c.xs[sp * RW + si], c.xs[sm * RW + si],
                               c.xs[sj * RW + si + 1], c.xs[sj * RW + si - 1], sA);
        }
        if (!row_in || cc < 0 || cc >= c.n) rv = T(0);
        rrow[si] = rv;
        if (c.lane == 2) pr_row(c.bp, 5, j)[si] = c.bs[sj * RW + si];  // b(j, c0+W) for the edge r'
    }
    named_bar_sync(1, (PR_NW + 1) * 32);
    const int f = j - 3;  // r' row of this step
    // ---------------- after the barrier: producer ------------------------------------------
    if (c.producer) {
        if (c.lane < 3) {
            // x'(j-1) at c0-1, c0+W, c0+W+1 (zero outside the interior)
            const int off = c.lane == 0 ? -1 : W + c.lane - 1;
            const int si = H + off, cc = c.c0 + off;
            T xv = T(0);
            if ((unsigned)(j - 1) < (unsigned)c.n && cc >= 0 && cc < c.n) {
                T acc = T(0);
                const int nt = tnt<T, S>(M);
#pragma unroll
                for (int t = 0; t < (S == SHAPE_GENERIC ? kMaxTerms : ShapeT<(S == SHAPE_GENERIC ? 1 : S)>::nt); ++t) {
                    if (S == SHAPE_GENERIC && t >= nt) break;
                    const T rv = pr_row(c.rr, 4, j - 1 + toff<T, S>(M, t, 0))[si + toff<T, S>(M, t, 1)];
                    acc = O::add(acc, O::mul(M.c[t], rv));
                }
                xv = relax<T>(FZ ? T(0) : c.xs[sm * RW + si], acc, sM, omega);
            }
            pr_row(c.xp, 4, j - 1)[si] = xv;
        } else if (c.lane == 3) {
            // r'(f) at column c0+W, and the strip-edge axis-0 weight on the top row of a group
            const int si = H + W, cc = c.c0 + W;
            T rv = T(0);
            if ((unsigned)f < (unsigned)c.n && cc < c.n) {
                const T* xf = pr_row(c.xp, 4, f);
                rv = residual2d<T>(pr_row(c.bp, 5, f)[si], xf[si], pr_row(c.xp, 4, f + 1)[si],
                                   pr_row(c.xp, 4, f - 1)[si], xf[si + 1], xf[si - 1], sA);
            }
            RE[ic] = rv;  // rows f (ic), f-1 (im), f-2 (ip)
            if ((f & 1) == 0) c.te[2 * PR_NW] = fw<T>(RE[ip], RE[im], RE[ic]);
        }
        __syncwarp();
        // stage j-1 was last read above: refill its slot with row j-1+ST
        if (c.lane == 0 && j - 1 + ST <= c.q_last) pr_issue<T, FZ>(c, j - 1 + ST, sm);
        return;
    }
    // ---------------- after the barrier: consumers -----------------------------------------
    // 1. full weighting of coarse row (j-6)/2 from the axis-0 weights of the previous step
    if (((j - 4) & 1) == 0) {
        const int I = (j - 6) >> 1;
        T tn = __shfl_down_sync(0xffffffffu, TP[0], 1);
        if (c.lane == 31) tn = c.te[2 * (c.warp + 1)];
        if (I >= c.I0 && I < c.I1) {
#pragma unroll
            for (int i = 0; i < VEC / 2; ++i) {
                const int J = (c.col >> 1) + i;
                const T t2 = 2 * i + 2 < VEC ? TP[2 * i + 2] : tn;
                if (J < c.m) c.crow0[(long long)I * c.cpx + i] = fw<T>(TP[2 * i], TP[2 * i + 1], t2);
            }
        }
    }
    // 2. x'(j-1) on the own columns
    RL[ic] = rrow[c.sidx - 1];
    RH[ic] = rrow[c.sidx + VEC];
    T out[VEC];
    const int nt = tnt<T, S>(M);
#pragma unroll
    for (int v = 0; v < VEC; ++v) {
        T acc = T(0);
#pragma unroll
        for (int t = 0; t < (S == SHAPE_GENERIC ? kMaxTerms : ShapeT<(S == SHAPE_GENERIC ? 1 : S)>::nt); ++t) {
            if (S == SHAPE_GENERIC && t >= nt) break;
            const T val = pick<T, VEC>(R[ip], R[im], R[ic], RL[ip], RL[im], RL[ic], RH[ip], RH[im], RH[ic],
                                       toff<T, S>(M, t, 0), toff<T, S>(M, t, 1), v);
            acc = O::add(acc, O::mul(M.c[t], val));
        }
        out[v] = relax<T>(FZ ? T(0) : X[im][v], acc, sM, omega);
    }
    if ((unsigned)(j - 1) >= (unsigned)c.n || c.last_strip) {
#pragma unroll
        for (int v = 0; v < VEC; ++v)
            if ((unsigned)(j - 1) >= (unsigned)c.n || c.col + v >= c.n) out[v] = T(0);  // x' exists on the interior
    }
    V16<T>::st(pr_row(c.xp, 4, j - 1) + c.sidx, out);
    if (j - 1 >= c.r0 && j - 1 < c.r_end) {
        T* dst = c.orow0 + (long long)(j - 1) * c.px;
        if (!c.last_strip || c.col + VEC <= c.n) {
            V16<T>::st(dst, out);
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (c.col + v < c.n) dst[v] = out[v];
        }
    }
    // 3. r'(f) = b - A x' on the own columns (x' rows f-1..f+1 were stored in earlier steps)
    {
        const T* xf = pr_row(c.xp, 4, f) + c.sidx;
        const T* xs1 = pr_row(c.xp, 4, f + 1) + c.sidx;
        const T* xn1 = pr_row(c.xp, 4, f - 1) + c.sidx;
        const T* bf = pr_row(c.bp, 5, f) + c.sidx;
        const bool f_in = (unsigned)f < (unsigned)c.n;
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            T rv = T(0);
            if (f_in && c.col + v < c.n) rv = residual2d<T>(bf[v], xf[v], xs1[v], xn1[v], xf[v + 1], xf[v - 1], sA);
            RP[ic][v] = rv;  // rows f (ic), f-1 (im), f-2 (ip)
        }
        // axis-0 weights on the top row of a coarse group (used next step)
        if ((f & 1) == 0) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) TP[v] = fw<T>(RP[ip][v], RP[im][v], RP[ic][v]);
            if (c.lane == 0) c.te[2 * c.warp] = TP[0];
        }
    }
}

template <class T, int S, bool FZ, bool NORM>
__global__ void __launch_bounds__((PR_NW + 1) * 32) k_sweep_rr2d(Layout L, Layout Lc, const T* __restrict__ x,
                                                                 const T* __restrict__ b, T* __restrict__ xo,
                                                                 T* __restrict__ bc, Terms<T> M, T sA, T sM, T omega,
                                                                 int rows, NormOut no) {
    using G = PRG<T>;
    constexpr int VEC = G::VEC;
    constexpr int W = G::W;
    constexpr int RW = G::RW;
    constexpr int ST = PR_ST;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    pdl_wait();
    pdl_trigger();
    PRCtx<T> c;
    c.xs = reinterpret_cast<T*>(smem_raw);
    c.bs = c.xs + ST * RW;
    c.rr = c.bs + ST * RW;
    c.xp = c.rr + 4 * RW;
    c.bp = c.xp + 4 * RW;
    c.te = c.bp + 5 * RW;
    c.full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(c.te + 2 * (PR_NW + 1)) + 15) & ~uintptr_t(15));
    c.warp = threadIdx.x >> 5;
    c.lane = threadIdx.x & 31;
    c.producer = c.warp == PR_NW;
    c.n = L.n;
    c.m = Lc.n;
    c.px = L.px;
    c.cpx = Lc.px;
    c.c0 = blockIdx.x * W;
    c.r0 = blockIdx.y * rows;  // rows is even
    c.r_end = min(c.r0 + rows, c.n);
    c.I0 = c.r0 >> 1;
    c.I1 = c.r_end == c.n ? c.m : (c.r_end >> 1);
    c.q0 = c.r0 - 3;              // first staged row (r from row r0-2)
    const int j_end = 2 * c.I1 + 4;  // last step: the full weighting of coarse row I1-1
    c.q_last = j_end + 1;
    c.last_strip = c.c0 + W > c.n;
    const int lc = (c.producer ? 0 : c.warp) * 32 + c.lane;
    c.sidx = PR_H + lc * VEC;
    c.col = c.c0 + lc * VEC;
    c.xrow0 = x + L.origin + (c.c0 - PR_H);
    c.brow0 = b + L.origin + (c.c0 - PR_H);
    c.orow0 = xo + L.origin + c.col;
    c.crow0 = bc + Lc.origin + (c.col >> 1);

    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; ++i) mbar_init(&c.full[i], 1);
        mbar_fence_init();
    }
    // rings start at zero (rows before the chunk's first computed row are read as zeros)
    for (int i = threadIdx.x; i < (4 + 4 + 5) * RW + 2 * (PR_NW + 1); i += blockDim.x) c.rr[i] = T(0);
    __syncthreads();
    if (c.producer && c.lane == 0)
        for (int q = c.q0; q < c.q0 + ST && q <= c.q_last; ++q) pr_issue<T, FZ>(c, q, q - c.q0);

    T X[3][VEC], R[3][VEC], RL[3], RH[3], RP[3][VEC], TP[VEC], RE[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        RL[i] = RH[i] = RE[i] = T(0);
#pragma unroll
        for (int v = 0; v < VEC; ++v) X[i][v] = R[i][v] = RP[i][v] = T(0);
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) TP[v] = T(0);
    mbar_wait(&c.full[0], 0);
    mbar_wait(&c.full[1], 0);
    if (!FZ && !c.producer) {
        V16<T>::ld(c.xs + 0 * RW + c.sidx, X[0]);  // x(q0)   = x(j-1) of step k = 1
        V16<T>::ld(c.xs + 1 * RW + c.sidx, X[1]);  // x(q0+1) = x(j)
    }
    double nacc = 0.0;
    const int K = j_end - c.q0;
    for (int kb = 0; kb <= K; kb += ST) {
        if (kb >= 1) pr_step<T, S, FZ, NORM, 0>(c, kb, X, R, RL, RH, RP, TP, RE, M, sA, sM, omega, nacc);
        if (kb + 1 <= K) pr_step<T, S, FZ, NORM, 1>(c, kb + 1, X, R, RL, RH, RP, TP, RE, M, sA, sM, omega, nacc);
        if (kb + 2 <= K) pr_step<T, S, FZ, NORM, 2>(c, kb + 2, X, R, RL, RH, RP, TP, RE, M, sA, sM, omega, nacc);
        if (kb + 3 <= K) pr_step<T, S, FZ, NORM, 3>(c, kb + 3, X, R, RL, RH, RP, TP, RE, M, sA, sM, omega, nacc);
        if (kb + 4 <= K) pr_step<T, S, FZ, NORM, 4>(c, kb + 4, X, R, RL, RH, RP, TP, RE, M, sA, sM, omega, nacc);
        if (kb + 5 <= K) pr_step<T, S, FZ, NORM, 5>(c, kb + 5, X, R, RL, RH, RP, TP, RE, M, sA, sM, omega, nacc);
    }
    if (NORM) norm_epilogue(nacc, no);
}

template <class T, int S, bool FZ, bool NORM>
static cudaError_t pr_launch(const Layout& L, const Layout& Lc, const T* x, const T* b, T* xo, T* bc,
                             const Terms<T>& M, T sA, T sM, T omega, const NormOut& no, cudaStream_t s) {
    using G = PRG<T>;
    constexpr int threads = (PR_NW + 1) * 32;
    cudaError_t e = cudaFuncSetAttribute(k_sweep_rr2d<T, S, FZ, NORM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)G::smem);
    if (e != cudaSuccess) return e;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep_rr2d<T, S, FZ, NORM>, threads, G::smem);
        if (occ <= 0) occ = 1;
    }
    const int strips = (L.n + G::W - 1) / G::W;
    int chunks = march_chunks(strips, num_sms() * occ, L.n, 16, 7);
    int rows = (L.n + chunks - 1) / chunks;
    rows += rows & 1;  // even: coarse rows partition across chunks
    chunks = (L.n + rows - 1) / rows;
    dim3 g(strips, chunks);
    return launch_pdl(k_sweep_rr2d<T, S, FZ, NORM>, g, dim3(threads), G::smem, s, L, Lc, x, b, xo, bc, M, sA, sM,
                      omega, rows, no);
}

template <class T, bool FZ, bool NORM>
static cudaError_t pr_shape(int shape, const Layout& L, const Layout& Lc, const T* x, const T* b, T* xo, T* bc,
                            const Terms<T>& M, T sA, T sM, T omega, const NormOut& no, cudaStream_t s) {
    switch (shape) {
        case SHAPE_C1: return pr_launch<T, SHAPE_C1, FZ, NORM>(L, Lc, x, b, xo, bc, M, sA, sM, omega, no, s);
        case SHAPE_STAR5: return pr_launch<T, SHAPE_STAR5, FZ, NORM>(L, Lc, x, b, xo, bc, M, sA, sM, omega, no, s);
        case SHAPE_BOX9: return pr_launch<T, SHAPE_BOX9, FZ, NORM>(L, Lc, x, b, xo, bc, M, sA, sM, omega, no, s);
        default: return pr_launch<T, SHAPE_GENERIC, FZ, NORM>(L, Lc, x, b, xo, bc, M, sA, sM, omega, no, s);
    }
}

// Opt-in (SPAIMG_PR=1): bitwise correct, but measured slower than the sweep + K2 pair on c2
// (0.444 vs 0.400 ms/cycle): at ~53 KB of shared memory (4 CTAs/SM) the march carries two
// extra dependent phases per row and stays latency-bound (measured/rejected).
bool sweep_rr_supported(const Layout& L) {
    const char* e = getenv("SPAIMG_PR");
    if (!(e && e[0] == '1')) return false;
    return L.dim == 2 && L.N > flat_threshold(2) && !getenv("SPAIMG_SWEEP_V1") && !getenv("SPAIMG_RESTRICT_V1");
}

template <class T>
cudaError_t launch_sweep_rr(const Layout& L, const Layout& Lc, const T* x, const T* b, T* xo, T* bc, const Terms<T>& M,
                            int shape, T sA, T sM, T omega, bool from_zero, cudaStream_t s, const NormOut* no) {
    const NormOut none{};
    if (no) {
        return from_zero ? pr_shape<T, true, true>(shape, L, Lc, x, b, xo, bc, M, sA, sM, omega, *no, s)
                         : pr_shape<T, false, true>(shape, L, Lc, x, b, xo, bc, M, sA, sM, omega, *no, s);
    }
    return from_zero ? pr_shape<T, true, false>(shape, L, Lc, x, b, xo, bc, M, sA, sM, omega, none, s)
                     : pr_shape<T, false, false>(shape, L, Lc, x, b, xo, bc, M, sA, sM, omega, none, s);
}

template cudaError_t launch_sweep_rr<double>(const Layout&, const Layout&, const double*, const double*, double*,
                                             double*, const Terms<double>&, int, double, double, double, bool,
                                             cudaStream_t, const NormOut*);
template cudaError_t launch_sweep_rr<float>(const Layout&, const Layout&, const float*, const float*, float*, float*,
                                            const Terms<float>&, int, float, float, float, bool, cudaStream_t,
                                            const NormOut*);

}  // namespace spaimg
