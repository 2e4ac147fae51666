// K1 2D row-marching sweep kernel (k_sweep2d_march) and its launcher, shared by the translation
// units that instantiate it: kernels_sweep.cu (plain / norm modes), kernels_sweep_pc.cu (K3 + K1)
// and kernels_sweep2.cu (two sweeps per march).  Split only to keep each unit's compile time
// down; see kernels_sweep.cu for the dispatch.
#pragma once

#include <cstdlib>

#include "kernels.h"
#include "march.cuh"
#include "ptx.cuh"

namespace spaimg {

// ------------------------------------------------------------------------------------------
// K1 2D: row-marching sweep.  A CTA owns a strip of W columns and a chunk of rows; one producer
// warp streams (x row, b row) pairs of the strip plus a VEC-wide halo into a ring of shared-
// memory stages with 1-D bulk copies (cp.async.bulk -> UBLKCP) completing on mbarriers.  Each
// consumer lane owns VEC = 16/sizeof(T) adjacent columns and keeps x(j-1..j+1) and r(j-2..j)
// of them in registers while marching down the rows; horizontal neighbours come from warp
// shuffles, warp-edge neighbours from a tiny shared edge ring, the two strip-halo residuals
// from the producer warp.  r is computed once per point; HBM traffic is x + b + x' (24 B/pt
// fp64) plus the (W+2VEC)/W column halo and the 4-row chunk priming, both L2 hits.
// ------------------------------------------------------------------------------------------
constexpr int M2_NW = 4;   // consumer warps per CTA
constexpr int M2_ST = 6;   // (x row, b row) ring depth; the step loop is unrolled by M2_ST

template <class T>
__host__ __device__ constexpr int m2_vec() { return 16 / (int)sizeof(T); }
template <class T>
__host__ __device__ constexpr int m2_width() { return 32 * m2_vec<T>() * M2_NW; }
template <class T>
__host__ __device__ constexpr int m2_rowlen() { return m2_width<T>() + 2 * m2_vec<T>(); }
// NM == 3 (prolongation + correction fused in front of the sweep): coarse correction rows
// [c0/2 - VEC, c0/2 + W/2 + VEC) staged in a ring indexed by coarse row
// ring depth: at step j the consumers read coarse rows fl2(j+3)-1 .. fl2(j+3) while the producer
// stages fl2(j+5), so 4 slots never alias a live row
constexpr int M2_CR = 4;  // must be a power of 2
// (TW strips start at c0 = bx (W - 2 VEC) - VEC, so the staged coarse row start is aligned down
// to a 16-byte boundary and the row is one VEC longer)
template <class T>
__host__ __device__ constexpr int m2_crowlen(bool two = false) { return m2_width<T>() / 2 + (two ? 3 : 2) * m2_vec<T>(); }
template <class T>
constexpr size_t m2_smem_bytes(bool pc = false, bool two = false) {
    return (size_t)2 * M2_ST * m2_rowlen<T>() * sizeof(T)   // x and b stages
           + (size_t)2 * m2_rowlen<T>() * sizeof(T)         // r rows (ring of 2)
           + (two ? (size_t)6 * m2_rowlen<T>() * sizeof(T) : 0)  // TW: x' rows (ring of 2), r' rows (ring of 4)
           + (pc ? (size_t)M2_CR * m2_crowlen<T>(two) * sizeof(T) : 0)  // coarse correction rows
           + (size_t)M2_ST * 8;                             // mbarriers
}


template <class T>
struct M2Ctx {
    T* xs;
    T* bs;
    T* rr;
    uint64_t* full;
    const T* xrow0;
    const T* brow0;
    T* orow0;  // output row 0, own first column
    long long px;
    int n, c0, col, sidx, q0, q_last, r0, r_end, lane;
    bool producer, last_strip;
    // TW: the second sweep's x' rows (ring of 2, horizontal neighbours) and r' rows (ring of 4)
    T* x1s;
    T* r2s;
    int tcons;        // consumer thread index 0 .. W/VEC-1
    // NM == 3: coarse correction e (multigrid.py:184) staged per coarse row
    T* es;            // ring of M2_CR coarse rows
    int crw;          // coarse row length in the ring (m2_crowlen)
    const T* erow0;   // coarse row 0 at coarse column c0/2 - VEC
    long long epx;
    int m, ce0;       // coarse interior size, first staged coarse column
    bool pc_edge;     // the strip (with its halo) holds coarse column 0 or m
};

__device__ __forceinline__ int fl2(int q) { return q >= 0 ? q / 2 : -((1 - q) / 2); }  // floor(q/2)

// x(q, .) += (P e)(q, .) on VEC staged columns starting at the even fine column k0 (staged
// index si): separable d-linear interpolation, axis 0 first, with the reference end formulas
// (multigrid.py:122-144) -- the k_prolong_correct2d tree.  Outside the interior P e is exactly
// 0 (zero frame), so halo columns/rows stay 0.
// EDGE = false: no first/last line of either axis is involved (warp-uniform fast path, no selects).
template <class T, bool EDGE>
__device__ __forceinline__ void m2_correct(const M2Ctx<T>& c, T* xrow, int q, int k0, int si) {
    constexpr int VEC = m2_vec<T>();
    const int CRW = c.crw;
    using O = Op<T>;
    auto row = [&](int cr) { return c.es + (cr & (M2_CR - 1)) * CRW - c.ce0; };  // M2_CR: power of 2
    // axis 0: t(J) at coarse columns J0-1 .. J0+VEC/2-1 (J0 = k0/2)
    const int J0 = k0 >> 1;
    T t[VEC / 2 + 1];
    if (q & 1) {
        const T* e0 = row((q - 1) >> 1) + J0 - 1;
#pragma unroll
        for (int i = 0; i <= VEC / 2; ++i) t[i] = e0[i];
    } else {
        const int I = q >> 1;
        const T* em = row(I - 1) + J0 - 1;
        const T* e0 = row(I) + J0 - 1;
#pragma unroll
        for (int i = 0; i <= VEC / 2; ++i) t[i] = pl_even<T>(em[i], e0[i], EDGE && I == 0, EDGE && I == c.m);
    }
    // axis 1: even column 2J -> pl_even(t(J-1), t(J)), odd column 2J+1 -> t(J)
    T xv[VEC];
    V16<T>::ld(xrow + si, xv);
#pragma unroll
    for (int i = 0; i < VEC / 2; ++i) {
        const int J = J0 + i;
        xv[2 * i] = O::add(xv[2 * i], pl_even<T>(t[i], t[i + 1], EDGE && J == 0, EDGE && J == c.m));
        xv[2 * i + 1] = O::add(xv[2 * i + 1], t[i + 1]);
    }
    V16<T>::st(xrow + si, xv);
}

// the whole staged x row q: every consumer its own columns, producer lanes 0 / 1 the strip halos
// (the producer warp is otherwise idle after the barrier, and a consumer warp doing them would
// run the correction twice)
template <class T>
__device__ __forceinline__ void m2_correct_row(const M2Ctx<T>& c, int q, int slot) {
    constexpr int VEC = m2_vec<T>();
    constexpr int W = m2_width<T>();
    constexpr int RW = m2_rowlen<T>();
    T* xrow = c.xs + slot * RW;
    // first/last lines: coarse row 0 / m on even fine rows, coarse column 0 / m inside the strip
    const bool edge = c.pc_edge || q <= 0 || q >= 2 * c.m;
    int k0 = c.col, si = c.sidx;
    if (c.producer) {
        if (c.lane >= 2) return;
        k0 = c.lane == 0 ? c.c0 - VEC : c.c0 + W;
        si = c.lane == 0 ? 0 : VEC + W;
    }
    if (edge)
        m2_correct<T, true>(c, xrow, q, k0, si);
    else
        m2_correct<T, false>(c, xrow, q, k0, si);
}

template <class T, int S, bool FZ, int NM = 0, bool TW = false>
__device__ __forceinline__ void m2_issue(const M2Ctx<T>& c, int q, int slot) {
    constexpr int RW = m2_rowlen<T>();
    constexpr uint32_t row_bytes = RW * sizeof(T);
    constexpr uint32_t crow_bytes = m2_crowlen<T>(TW) * sizeof(T);
    // NM == 3: fine row q brings the coarse row floor(q/2) it is the first to need (the first
    // staged row also brings the row below)
    const int ncr = NM == 3 ? ((q & 1) == 0 || q == c.q0 ? 1 : 0) + (q == c.q0 && (q & 1) == 0 ? 1 : 0) : 0;
    // TW stages rows up to 4 past the chunk; rows beyond the two-row zero frame are loaded from
    // the frame (their values only feed results forced to zero outside the interior)
    const int qr = TW ? min(max(q, -kGhost), c.n - 1 + kGhost) : q;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&c.full[slot], (FZ ? row_bytes : 2 * row_bytes) + ncr * crow_bytes);
    if (!FZ) bulk_g2s(c.xs + slot * RW, c.xrow0 + (long long)qr * c.px, row_bytes, &c.full[slot]);
    bulk_g2s(c.bs + slot * RW, c.brow0 + (long long)qr * c.px, row_bytes, &c.full[slot]);
    if constexpr (NM == 3) {
        for (int i = 0; i < ncr; ++i) {
            const int cr = fl2(q) - i;
            const int crr = TW ? min(max(cr, -kGhost), c.m - 1 + kGhost) : cr;
            bulk_g2s(c.es + ((cr % M2_CR + M2_CR) % M2_CR) * m2_crowlen<T>(TW), c.erow0 + (long long)crr * c.epx,
                     crow_bytes, &c.full[slot]);
        }
    }
}

// TW (two sweeps in one march): registers of the second sweep, rings indexed by step mod 6/3
// (r' rows live in shared memory, read back with their neighbours: fewer registers per thread)
template <class T> struct M2Two {
    T X1[6][m2_vec<T>()];  // x' rows (own columns)
    T B[3][m2_vec<T>()];   // b rows (the stage ring has moved on when the second sweep needs them)
};

// One marching step k (row j = q0 + k): r(j) for the strip (+ halo), then output row j-1.
// P = k mod 6 makes every stage slot and register-row index a compile-time constant.  PROD: the
// producer warp's step (the march loop is instantiated per role, so no step tests the role);
// EDGE: the strip holds columns outside the interior (column masks compiled in).  orow: the
// output row pointer of this step (row j-1, own first column), advanced by every step.
template <class T, int S, bool FZ, int NM, int P, bool TW, bool PROD, bool EDGE>
__device__ __forceinline__ void m2_step(const M2Ctx<T>& c, int k, T (&X)[3][m2_vec<T>()], T (&R)[3][m2_vec<T>()],
                                        T (&RL)[3], T (&RH)[3], M2Two<T>& tw, const Terms<T>& M, T sA, T sM, T omega,
                                        double& nacc, T*& orow) {
    using O = Op<T>;
    constexpr int VEC = m2_vec<T>();
    constexpr int W = m2_width<T>();
    constexpr int RW = m2_rowlen<T>();
    constexpr int ST = M2_ST;
    constexpr int sj = P % ST, sp = (P + 1) % ST, sm = (P + ST - 1) % ST;  // stage slots of rows j, j+1, j-1
    constexpr int ic = P % 3, ip = (P + 1) % 3, im = (P + 2) % 3;          // register rows j, j+1, j-1
    constexpr int rs = P % 2;                                               // r row ring slot
    const int j = c.q0 + k;
    mbar_wait(&c.full[sp], (uint32_t)(((k + 1) / ST) & 1));
    const bool row_in = (unsigned)j < (unsigned)c.n;
    T* rrow = c.rr + rs * RW;
    T* const dst = orow;
    orow += c.px;
    if constexpr (!PROD) {
        T bj[VEC];
        V16<T>::ld(c.bs + sj * RW + c.sidx, bj);
        if constexpr (TW) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) tw.B[P % 3][v] = bj[v];
        }
        if constexpr (FZ) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) R[ic][v] = bj[v];  // b - A 0 == b exactly
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
        if constexpr (EDGE) {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (!row_in || c.col + v >= c.n || (TW && c.col + v < 0)) R[ic][v] = T(0);  // r is zero outside
        } else if (!row_in) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) R[ic][v] = T(0);
        }
        // ||r||^2 of own rows (TW: strips overlap by VEC columns; the edge consumers do not count)
        if ((NM == 1 || NM == 2) && j >= c.r0 && j < c.r_end && (!TW || (c.tcons > 0 && c.tcons < W / VEC - 1))) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) nacc += (double)R[ic][v] * (double)R[ic][v];  // ||r||^2, own rows
        }
        if (NM != 2) V16<T>::st(rrow + c.sidx, R[ic]);
    } else if (NM != 2 && c.lane < 2) {  // PROD
        // strip-halo residuals at columns c0-1 (lane 0) and c0+W (lane 1)
        const int si = c.lane == 0 ? VEC - 1 : VEC + W;
        const int cc = c.lane == 0 ? c.c0 - 1 : c.c0 + W;
        T rv;
        if constexpr (FZ) {
            rv = c.bs[sj * RW + si];
        } else {
            rv = residual2d<T>(c.bs[sj * RW + si], c.xs[sj * RW + si], c.xs[sp * RW + si], c.xs[sm * RW + si],
                               c.xs[sj * RW + si + 1], c.xs[sj * RW + si - 1], sA);
        }
        if (!row_in || cc < 0 || cc >= c.n) rv = T(0);
        rrow[si] = rv;
    }
    named_bar_sync(1, (M2_NW + 1) * 32);
    if constexpr (PROD) {
        // stage j-1 was last read before this barrier: refill its slot with row j-1+ST
        if (c.lane == 0 && j - 1 + ST <= c.q_last) m2_issue<T, S, FZ, NM, TW>(c, j - 1 + ST, sm);
        if constexpr (NM == 3) {  // the strip halos of row j+3 (see m2_correct_row)
            constexpr int s3 = (P + 3) % ST;
            if (j + 3 <= c.q_last) {
                mbar_wait(&c.full[s3], (uint32_t)(((k + 3) / ST) & 1));
                m2_correct_row<T>(c, j + 3, s3);
            }
        }
        return;
    }
    if (NM == 2) return;
    if constexpr (NM == 3) {
        // x + P e of row j+3 (read from step k+2 on, i.e. after the next barrier)
        constexpr int s3 = (P + 3) % ST;
        if (j + 3 <= c.q_last) {
            mbar_wait(&c.full[s3], (uint32_t)(((k + 3) / ST) & 1));
            m2_correct_row<T>(c, j + 3, s3);
        }
    }
    RL[ic] = rrow[c.sidx - 1];
    RH[ic] = rrow[c.sidx + VEC];
    if (j - 1 < c.r0 - (TW ? 2 : 0)) return;
    // output row j-1: r rows j-2 (R[ip]), j-1 (R[im]), j (R[ic])
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
    if constexpr (!TW) {
        if (!EDGE || c.col + VEC <= c.n) {
            V16<T>::st(dst, out);
        } else {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (c.col + v < c.n) dst[v] = out[v];
        }
    } else {
        // ---- second sweep (TW), three rows behind the first, bitwise the same trees ----------
        // x'(j-1): zero outside the interior (the reference's zero extension of the new iterate)
        constexpr int k1 = (P + 5) % 6, k2 = (P + 4) % 6, k3 = (P + 3) % 6, k4 = (P + 2) % 6;
        const bool rin1 = (unsigned)(j - 1) < (unsigned)c.n;
#pragma unroll
        for (int v = 0; v < VEC; ++v)
            tw.X1[k1][v] = (rin1 && (unsigned)(c.col + v) < (unsigned)c.n) ? out[v] : T(0);
        V16<T>::st(c.x1s + ((P + 1) & 1) * RW + c.sidx, tw.X1[k1]);
        // r'(j-2) = b(j-2) - A x' on rows j-3..j-1 (x'(j-2)'s neighbours: written last step)
        if (j - 2 >= c.r0 - 1) {
            T r2[VEC];
            const T* xr = c.x1s + (P & 1) * RW;
            const T left = xr[c.sidx - 1], right = xr[c.sidx + VEC];
            const bool rin2 = (unsigned)(j - 2) < (unsigned)c.n;
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                const T xe = v + 1 < VEC ? tw.X1[k2][v + 1] : right;
                const T xw = v > 0 ? tw.X1[k2][v - 1] : left;
                const T rv = residual2d<T>(tw.B[(P + 1) % 3][v], tw.X1[k2][v], tw.X1[k1][v], tw.X1[k3][v], xe, xw, sA);
                r2[v] = (rin2 && (unsigned)(c.col + v) < (unsigned)c.n) ? rv : T(0);
            }
            V16<T>::st(c.r2s + ((j - 2) & 3) * RW + c.sidx, r2);
        }
        // x''(j-4) = x'(j-4) + omega (M r') sM from r' rows j-5..j-3 (shared ring, written in the
        // three previous steps)
        if (j - 4 >= c.r0 && j - 4 < c.r_end) {
            T ra[VEC], rb[VEC], rc2[VEC];
            const T* p5 = c.r2s + ((j - 5) & 3) * RW + c.sidx;
            const T* p4 = c.r2s + ((j - 4) & 3) * RW + c.sidx;
            const T* p3 = c.r2s + ((j - 3) & 3) * RW + c.sidx;
            V16<T>::ld(p5, ra);
            V16<T>::ld(p4, rb);
            V16<T>::ld(p3, rc2);
            const T l5 = p5[-1], l4 = p4[-1], l3 = p3[-1], h5 = p5[VEC], h4 = p4[VEC], h3 = p3[VEC];
            T out2[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                T acc = T(0);
#pragma unroll
                for (int t = 0; t < (S == SHAPE_GENERIC ? kMaxTerms : ShapeT<(S == SHAPE_GENERIC ? 1 : S)>::nt); ++t) {
                    if (S == SHAPE_GENERIC && t >= nt) break;
                    const T val = pick<T, VEC>(ra, rb, rc2, l5, l4, l3, h5, h4, h3, toff<T, S>(M, t, 0),
                                               toff<T, S>(M, t, 1), v);
                    acc = O::add(acc, O::mul(M.c[t], val));
                }
                out2[v] = relax<T>(tw.X1[k4][v], acc, sM, omega);
            }
            // strips overlap by VEC columns on each side: the edge consumers only feed their neighbours
            if (c.tcons > 0 && c.tcons < W / VEC - 1) {
                T* dst2 = dst - 3 * c.px;  // row j-4
                if (c.col + VEC <= c.n) {
                    V16<T>::st(dst2, out2);
                } else {
#pragma unroll
                    for (int v = 0; v < VEC; ++v)
                        if (c.col + v < c.n) dst2[v] = out2[v];
                }
            }
        }
    }
}

template <class T, int S, bool FZ, int NM, bool TW = false>
__global__ void __launch_bounds__((M2_NW + 1) * 32, TW ? 3 : (NM == 3 ? 5 : 1)) k_sweep2d_march(Layout L, const T* __restrict__ x,
                                                                     const T* __restrict__ b, T* __restrict__ xo,
                                                                     Terms<T> M, T sA, T sM, T omega, int rows,
                                                                     NormOut no, const T* __restrict__ e, Layout Lc) {
    constexpr int VEC = m2_vec<T>();
    constexpr int W = m2_width<T>();
    constexpr int RW = m2_rowlen<T>();
    constexpr int ST = M2_ST;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    M2Ctx<T> c;
    c.xs = reinterpret_cast<T*>(smem_raw);
    c.bs = c.xs + ST * RW;
    c.rr = c.bs + ST * RW;
    c.x1s = c.rr + 2 * RW;
    c.r2s = c.x1s + 2 * RW;
    c.es = c.rr + (TW ? 8 : 2) * RW;
    c.full = reinterpret_cast<uint64_t*>(c.es + (NM == 3 ? M2_CR * m2_crowlen<T>(TW) : 0));
    c.crw = m2_crowlen<T>(TW);
    const int warp = threadIdx.x >> 5;
    c.lane = threadIdx.x & 31;
    c.producer = warp == M2_NW;
    c.n = L.n;
    c.px = L.px;
    // TW: strips of W columns overlapping by VEC on each side, W - 2 VEC output columns each
    c.c0 = TW ? (int)blockIdx.x * (W - 2 * VEC) - VEC : (int)blockIdx.x * W;
    c.r0 = blockIdx.y * rows;
    const int r_end = min(c.r0 + rows, c.n);
    c.r_end = r_end;
    c.q0 = c.r0 - (TW ? 4 : 2);        // first staged row
    c.q_last = r_end + (TW ? 4 : 1);   // last staged row
    c.last_strip = c.c0 + W > c.n;
    c.tcons = (c.producer ? 0 : warp) * 32 + c.lane;
    c.sidx = VEC + (c.producer ? 0 : warp) * 32 * VEC + c.lane * VEC;
    c.col = c.c0 + (c.producer ? 0 : warp) * 32 * VEC + c.lane * VEC;
    c.xrow0 = x + L.origin + (c.c0 - VEC);
    c.brow0 = b + L.origin + (c.c0 - VEC);
    c.orow0 = xo + L.origin + c.col;
    if constexpr (NM == 3) {
        // first staged coarse column, aligned down to 16 bytes (floor division: c0 < 0 on strip 0)
        const int ce = c.c0 / 2 - VEC;
        c.ce0 = TW ? (ce >= 0 ? ce / VEC : -((-ce + VEC - 1) / VEC)) * VEC : ce;
        c.erow0 = e + Lc.origin + c.ce0;
        c.epx = Lc.px;
        c.m = Lc.n;
        c.pc_edge = c.c0 - VEC <= 0 || ((c.c0 + W + VEC) >> 1) >= Lc.n;
    }

    if (threadIdx.x == 0) {
        for (int i = 0; i < ST; ++i) mbar_init(&c.full[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (c.producer && c.lane == 0)
        for (int q = c.q0; q < c.q0 + ST && q <= c.q_last; ++q) m2_issue<T, S, FZ, NM, TW>(c, q, q - c.q0);

    T X[3][VEC], R[3][VEC], RL[3], RH[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        RL[i] = RH[i] = T(0);
#pragma unroll
        for (int v = 0; v < VEC; ++v) X[i][v] = R[i][v] = T(0);
    }
    mbar_wait(&c.full[0], 0);
    mbar_wait(&c.full[1], 0);
    if constexpr (NM == 3) {  // rows q0 .. q0+3 corrected before the march (then 2 steps ahead)
        for (int i = 0; i < 4 && c.q0 + i <= c.q_last; ++i) {
            mbar_wait(&c.full[i], 0);
            m2_correct_row<T>(c, c.q0 + i, i);
        }
        __syncthreads();
    }
    if (!FZ && !c.producer) {
        V16<T>::ld(c.xs + 0 * RW + c.sidx, X[0]);  // x(q0)   = x(j-1) of step k = 1
        V16<T>::ld(c.xs + 1 * RW + c.sidx, X[1]);  // x(q0+1) = x(j)
    }
    double nacc = 0.0;
    M2Two<T> tw;
    // steps k = 1 .. K: rows j = q0+1 .. r_end (+3 with TW, whose second sweep trails by 3 rows)
    const int K = r_end + (TW ? 3 : 0) - c.q0;
    T* orow = c.orow0 + (long long)c.q0 * c.px;  // step k = 1 writes row j-1 = q0
    // one march loop per role (and, for the consumers, per strip kind), so that no step tests
    // the role or carries column masks it does not need
#define M2_MARCH(PROD, EDGE)                                                                                    \
    for (int kb = 0; kb <= K; kb += ST) {                                                                       \
        if (kb >= 1) m2_step<T, S, FZ, NM, 0, TW, PROD, EDGE>(c, kb, X, R, RL, RH, tw, M, sA, sM, omega, nacc, orow);         \
        if (kb + 1 <= K) m2_step<T, S, FZ, NM, 1, TW, PROD, EDGE>(c, kb + 1, X, R, RL, RH, tw, M, sA, sM, omega, nacc, orow); \
        if (kb + 2 <= K) m2_step<T, S, FZ, NM, 2, TW, PROD, EDGE>(c, kb + 2, X, R, RL, RH, tw, M, sA, sM, omega, nacc, orow); \
        if (kb + 3 <= K) m2_step<T, S, FZ, NM, 3, TW, PROD, EDGE>(c, kb + 3, X, R, RL, RH, tw, M, sA, sM, omega, nacc, orow); \
        if (kb + 4 <= K) m2_step<T, S, FZ, NM, 4, TW, PROD, EDGE>(c, kb + 4, X, R, RL, RH, tw, M, sA, sM, omega, nacc, orow); \
        if (kb + 5 <= K) m2_step<T, S, FZ, NM, 5, TW, PROD, EDGE>(c, kb + 5, X, R, RL, RH, tw, M, sA, sM, omega, nacc, orow); \
    }
    if (c.producer) {
        M2_MARCH(true, true)
    } else if (TW || c.last_strip) {
        M2_MARCH(false, true)
    } else {
        if constexpr (!TW) {
            M2_MARCH(false, false)
        }
    }
#undef M2_MARCH
    if (NM == 1 || NM == 2) norm_epilogue(nacc, no);
}

template <class T, int S, bool FZ, int NM, bool TW = false>
static cudaError_t launch_sweep2d_march(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA,
                                        T sM, T omega, const NormOut& no, cudaStream_t s, const T* e = nullptr,
                                        const Layout* Lc = nullptr) {
    constexpr size_t smem = m2_smem_bytes<T>(NM == 3, TW);
    if (smem > 48 * 1024) {  // per device, so set on every launch (host-side, cheap)
        cudaError_t err = cudaFuncSetAttribute(k_sweep2d_march<T, S, FZ, NM, TW>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (err != cudaSuccess) return err;
    }
    constexpr int threads = (M2_NW + 1) * 32;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep2d_march<T, S, FZ, NM, TW>, threads, smem);
        if (occ <= 0) occ = 1;
    }
    const int W = m2_width<T>();
    const int Wout = TW ? W - 2 * m2_vec<T>() : W;
    const int strips = (L.n + Wout - 1) / Wout;
    const int slots = num_sms() * occ;
    int chunks = march_chunks(strips, slots, L.n, 16, TW ? 8 : 4);
    const int rows = (L.n + chunks - 1) / chunks;
    chunks = (L.n + rows - 1) / rows;
    dim3 g(strips, chunks);
    return launch_k(k_sweep2d_march<T, S, FZ, NM, TW>, g, dim3(threads), smem, s, L, x, b, xo, M, sA, sM, omega,
                    rows, no, e, Lc ? *Lc : L);
}

}  // namespace spaimg
