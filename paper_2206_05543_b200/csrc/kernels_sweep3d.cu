// K1 3D: plane-marching fused SPAI sweep (x' = x + omega M (b - A x), reference
// multigrid.py:98-100) with TMA tensor-tile staging.
//
// A CTA owns a TY x TX tile of (axis1, axis2) and marches along axis 0 over a chunk of planes.
// Thread 0 streams, per plane, the x tile with a 2-row / VEC-column halo and the b tile with a
// 1-row halo into a 4-deep ring of shared-memory stages with cp.async.bulk.tensor.3d (SASS
// UTMALDG) completing on mbarriers.  Each thread owns 2 rows x VEC columns and keeps
// x(j-1..j+1) and r(j-2..j) of them in registers (register-blocked z-marching); r(j) of the
// tile plus its one-point ring goes to a 3-plane shared ring from which M takes its in-plane
// neighbours.  r is computed once per tile point (the ring is recomputed by the neighbour
// tile: 2(TX+TY)/(TX*TY) extra).  The step loop is unrolled by 3 so the register-array and
// r-ring indices are compile-time constants; the stage slots (k mod 4) are runtime.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

#include "kernels.h"
#include "march.cuh"
#include "ptx.cuh"

namespace spaimg {

constexpr int M3_TY = 16;  // tile rows (axis 1)
constexpr int M3_NW = 8;   // warps; each owns 2 tile rows
constexpr int M3_ST = 4;   // TMA stage ring depth
constexpr int M3_RR = 3;   // r plane ring depth
constexpr int M3_THREADS = M3_NW * 32;

template <class T> struct M3 {
    static constexpr int VEC = 16 / (int)sizeof(T);
    static constexpr int TX = 32 * VEC;            // tile columns (axis 2)
    static constexpr int TY = M3_TY;
    static constexpr int RW = TX + 2 * VEC;        // staged row length
    static constexpr int XR = TY + 4;              // x stage rows  [y0-2, y0+TY+2)
    static constexpr int BR = TY + 2;              // b stage rows  [y0-1, y0+TY+1)
    static constexpr int RR = TY + 2;              // r plane rows  [y0-1, y0+TY+1)
    static constexpr int al(int e) { return (e * (int)sizeof(T) + 127) / 128 * 128 / (int)sizeof(T); }
    static constexpr int XS = al(XR * RW);         // elements per x stage (128-B multiple)
    static constexpr int BS = al(BR * RW);
    static constexpr int RS = al(RR * RW);
    static constexpr int NRING = 2 * TX + 2 * TY + 4;
    static constexpr int NRP = (NRING + M3_THREADS - 1) / M3_THREADS;  // ring points per thread
    // NM == 4 (K3 + K1: prolongation + correction fused in front of the sweep): the staged coarse
    // correction tile, rows [y0/2 - 2, y0/2 + TY/2 + 1), columns [x0/2 - VEC, x0/2 + TX/2 + VEC): the
    // first column needed is x0/2 - VEC/2 - 1; the tile starts on a 16-byte boundary (TMA box
    // start addresses that are not 16-byte aligned fault)
    static constexpr int ECW = TX / 2 + 2 * VEC;   // staged coarse row length (16-byte multiple)
    static constexpr int ER = TY / 2 + 3;          // staged coarse rows
    static constexpr int ES = al(ER * ECW);
    static constexpr int EST = 3;                  // coarse plane ring (indexed by coarse plane mod 3)
    static __device__ __forceinline__ int eslot(int I) { return (I + 3 * (1 << 20)) % EST; }
    static constexpr int NHALO = 2 * (TX / VEC + 2) + 2 * (TY / 2);  // 2 x VEC blocks of the x stage's halo
};

// Shared-memory plan per mode.  The K3 + K1 variant corrects plane j+2 in step j, so three x
// stages are live and a fourth would leave nothing in flight; instead every thread keeps x(j-1) of
// its ring point in a register, which frees x(j)'s stage right after step j's barrier: x(j+4) is
// issued then (two steps of lead, as in the plain sweep).  b(j) is read only in step j and rides
// with x(j+1) (so the last staged x plane brings the last b needed): three b stages.
template <class T, int NM> struct M3S {
    using G = M3<T>;
    static constexpr bool PC = NM == 4;
    static constexpr int BST = PC ? 3 : M3_ST;   // b stage ring
    static constexpr int RRD = M3_RR;            // r plane ring
    static constexpr size_t smem =
        (size_t)(M3_ST * G::XS + BST * G::BS + RRD * G::RS + (PC ? G::EST * G::ES : 0)) * sizeof(T) + M3_ST * 8;
};

template <class T>
struct M3Ctx {
    T* xs;
    T* bs;
    T* rr;
    uint64_t* full;
    T* obase;  // output at (plane 0, own row 0, own column)
    long long px, pp;
    int n, x0, y0, q0, q_last, z0, z_end, yl, xl, tid;
    bool edge;  // tile touches the right/bottom boundary (masking needed)
    // this thread's ring point(s): offset in an r plane / b stage (an x stage: + RW), -1 = none;
    // inside the interior in-plane
    int rro[M3<T>::NRP];
    bool rin[M3<T>::NRP];
    int cx, cy;  // TMA coordinates of the tile's stage origin (x stage)
    int ghost;   // the layout's ghost planes/rows (TMA coordinate of interior 0)
    // NM == 3 (K2 residual + restriction): coarse output level
    T* cb;
    long long cpx, cpp, corg;
    int cm;
    // NM == 4 (K3 + K1): coarse correction e (multigrid.py:184) staged per coarse plane
    T* es;
    int ecx, ecy, eghost;  // TMA coordinates of the staged coarse tile's origin; coarse ghost planes
    bool pc_edge;          // the tile (with its halo) touches a first/last line of axis 1 or 2
    // the thread's own block [0] and its halo block [1] (threads < NHALO): tile-local first row /
    // column, offset in an x stage, offset of coarse (Y-1, X-1) in a staged coarse plane
    int pry[2], prx[2], pxo[2], peo[2];
};

// K2 output of coarse plane I = (j-2)/2 from r planes j-2, j-1, j: full weighting along axis 0,
// then axis 1, then axis 2 (multigrid.py:104-119), the k_restrict tree.  Warp w owns coarse row
// y0/2 + w and each lane VEC/2 coarse columns: the axis-0 weights of its own 2 x VEC fine points
// come from the r registers, fine row 2w+2 from the shared r planes, and the column to the right
// from the next lane (the last lane reads the shared ring column).
template <class T>
__device__ __forceinline__ void m3_restrict_out(const M3Ctx<T>& c, int j, const T* r0, const T* r1, const T* r2,
                                                const T (&Rj)[2][M3<T>::VEC], const T (&Rj1)[2][M3<T>::VEC],
                                                const T (&Rj2)[2][M3<T>::VEC]) {
    using G = M3<T>;
    constexpr int VEC = G::VEC;
    constexpr int RW = G::RW;
    const int I = (j - 2) >> 1;
    const int lane = c.tid & 31;
    T t[3][VEC + 1];
#pragma unroll
    for (int yy = 0; yy < 2; ++yy)
#pragma unroll
        for (int v = 0; v < VEC; ++v) t[yy][v] = fw<T>(Rj2[yy][v], Rj1[yy][v], Rj[yy][v]);
    const int s2 = (c.yl + 3) * RW + VEC + c.xl;  // fine row yl+2 (the next warp's / ring row)
#pragma unroll
    for (int v = 0; v < VEC; ++v) t[2][v] = fw<T>(r2[s2 + v], r1[s2 + v], r0[s2 + v]);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        t[a][VEC] = __shfl_down_sync(0xffffffffu, t[a][0], 1);
        if (lane == 31) {
            const int sa = (c.yl + a + 1) * RW + VEC + c.xl + VEC;
            t[a][VEC] = fw<T>(r2[sa], r1[sa], r0[sa]);
        }
    }
    const int Y = (c.y0 >> 1) + (c.yl >> 1);
#pragma unroll
    for (int i = 0; i < VEC / 2; ++i) {
        const int X = (c.x0 >> 1) + (c.xl >> 1) + i;
        T u[3];
#pragma unroll
        for (int qk = 0; qk < 3; ++qk) u[qk] = fw<T>(t[0][2 * i + qk], t[1][2 * i + qk], t[2][2 * i + qk]);
        if (Y < c.cm && X < c.cm) c.cb[c.corg + (long long)I * c.cpp + (long long)Y * c.cpx + X] = fw<T>(u[0], u[1], u[2]);
    }
}

// stage plane q on full[slot]: x(q) into x slot `slot`, b into its own ring, and (K3 + K1) the
// coarse correction plane(s) fine plane q is the first to need
template <class T, bool FZ, int NM>
__device__ __forceinline__ void m3_issue(const M3Ctx<T>& c, const CUtensorMap* xm, const CUtensorMap* bm,
                                         const CUtensorMap* em, int q, int slot) {
    using G = M3<T>;
    using SP = M3S<T, NM>;
    constexpr uint32_t xb = G::XR * G::RW * sizeof(T), bb = G::BR * G::RW * sizeof(T);
    constexpr uint32_t eb = G::ER * G::ECW * sizeof(T);
    // K3 + K1: b(q-1) rides with x(q) (x(q) is waited for in step q-2, b(q-1) is read in step q-1
    // alone); r starts at plane q0+1, so the first two staged planes bring no b
    const int qb = SP::PC ? q - 1 : q;
    const bool with_b = !SP::PC || qb > c.q0;
    const int bslot = SP::PC ? (qb - c.q0 - 1) % 3 : slot;  // b(q0 + 1 + i) in slot i % 3
    // fine plane q brings the coarse plane floor(q/2) it is the first to need (the first staged
    // plane also the one below when q is even)
    const int ncr = SP::PC ? ((q & 1) == 0 || q == c.q0 ? 1 : 0) + (q == c.q0 && (q & 1) == 0 ? 1 : 0) : 0;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&c.full[slot], (FZ ? 0 : xb) + (with_b ? bb : 0) + ncr * eb);
    if (!FZ) tma_load_3d(c.xs + slot * G::XS, xm, c.cx, c.cy, c.ghost + q, &c.full[slot]);
    if (with_b) tma_load_3d(c.bs + bslot * G::BS, bm, c.cx, c.cy + 1, c.ghost + qb, &c.full[slot]);
    if constexpr (SP::PC) {
        for (int i = 0; i < ncr; ++i) {
            const int I = (q >> 1) - i;  // arithmetic shift: floor(q/2)
            tma_load_3d(c.es + G::eslot(I) * G::ES, em, c.ecx, c.ecy, c.eghost + I, &c.full[slot]);
        }
    }
}

// K3 + K1: x(q, .) += (P e)(q, .) on the 2 x VEC block of the staged x plane at tile-local fine
// rows ry, ry+1 (ry even, -2 .. TY) and columns rx .. rx+VEC-1 (rx a multiple of VEC, -VEC .. TX):
// separable d-linear interpolation, axis 0 first, then 1, then 2, with the reference end formulas
// (multigrid.py:122-144) -- the k_prolong_correct3d tree.  Outside the interior P e is exactly 0
// (zero frames), so the halo of a boundary tile stays 0.  EDGE = false: no first/last line of
// any axis is involved (warp-uniform fast path, no selects).
template <class T, bool EDGE>
__device__ __forceinline__ void m3_correct(const M3Ctx<T>& c, T* xr, const T* em, const T* e0, int q, int ry, int rx) {
    using G = M3<T>;
    using O = Op<T>;
    constexpr int VEC = G::VEC, C = VEC / 2, ECW = G::ECW;
    const int m = c.cm;
    // em / e0: the staged coarse planes floor(q/2) - 1 and floor(q/2) at coarse (Y-1, X-1) of the
    // block's first cell
    T t[2][C + 1];
    if (q & 1) {
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
            for (int i = 0; i <= C; ++i) t[d][i] = e0[d * ECW + i];
    } else {
        const int I = q >> 1;
        const bool fI = EDGE && I == 0, lI = EDGE && I == m;
#pragma unroll
        for (int d = 0; d < 2; ++d)
#pragma unroll
            for (int i = 0; i <= C; ++i) t[d][i] = pl_even<T>(em[d * ECW + i], e0[d * ECW + i], fI, lI);
    }
    const int J = (c.y0 + ry) >> 1, K0 = (c.x0 + rx) >> 1;
    const bool fJ = EDGE && J == 0, lJ = EDGE && J == m;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        T u[C + 1];
#pragma unroll
        for (int i = 0; i <= C; ++i) u[i] = h ? t[1][i] : pl_even<T>(t[0][i], t[1][i], fJ, lJ);
        T xv[VEC];
        V16<T>::ld(xr + h * G::RW, xv);
#pragma unroll
        for (int i = 0; i < C; ++i) {
            const int K = K0 + i;
            xv[2 * i] = O::add(xv[2 * i], pl_even<T>(u[i], u[i + 1], EDGE && K == 0, EDGE && K == m));
            xv[2 * i + 1] = O::add(xv[2 * i + 1], u[i + 1]);
        }
        V16<T>::st(xr + h * G::RW, xv);
    }
}

// tile-local (first row, first column) of halo block h of the x stage (0 .. NHALO-1)
template <class T>
__device__ __forceinline__ void m3_halo_block(int h, int& ry, int& rx) {
    using G = M3<T>;
    constexpr int VEC = G::VEC, NBX = G::TX / VEC + 2;
    if (h < 2 * NBX) {
        ry = h < NBX ? -2 : G::TY;
        rx = ((h < NBX ? h : h - NBX) - 1) * VEC;
    } else {
        const int g = h - 2 * NBX;
        ry = (g % (G::TY / 2)) * 2;
        rx = g < G::TY / 2 ? -VEC : G::TX;
    }
}

// the whole staged x plane q in `slot`, in place: every thread its own 2 x VEC block, the first
// NHALO threads also one block of the halo frame (the blocks' stage offsets are per-thread
// constants, M3Ctx::pxo / peo)
// es0: the ring slot of coarse plane floor(q/2) (the plane an odd q copies, the upper plane of an
// even q); the plane below is one slot back
template <class T>
__device__ __forceinline__ void m3_correct_plane(const M3Ctx<T>& c, int q, int slot, int es0) {
    using G = M3<T>;
    T* xpl = c.xs + slot * G::XS;
    // first/last lines: coarse plane 0 / m on even fine planes, and the tile's own edge flag
    const bool edge = c.pc_edge || q <= 0 || q >= 2 * c.cm;
    const T* e0 = c.es + es0 * G::ES;
    const T* em = c.es + (es0 == 0 ? G::EST - 1 : es0 - 1) * G::ES;
    const bool halo = c.tid < G::NHALO;
    if (edge) {
        m3_correct<T, true>(c, xpl + c.pxo[0], em + c.peo[0], e0 + c.peo[0], q, c.pry[0], c.prx[0]);
        if (halo) m3_correct<T, true>(c, xpl + c.pxo[1], em + c.peo[1], e0 + c.peo[1], q, c.pry[1], c.prx[1]);
    } else {
        m3_correct<T, false>(c, xpl + c.pxo[0], em + c.peo[0], e0 + c.peo[0], q, 0, 0);
        if (halo) m3_correct<T, false>(c, xpl + c.pxo[1], em + c.peo[1], e0 + c.peo[1], q, 0, 0);
    }
    fence_proxy_async_smem();  // the slot is refilled by TMA later
}

// r at this thread's ring point (stage offset ro) of plane j.  CACHE (every mode that stages x):
// x(j-1) at the point comes from `prev` (this thread read it as x(j) a step ago), so x(j-1)'s
// stage is not touched and can be refilled a step earlier; prev is then advanced to x(j).
template <class T, bool FZ, bool CACHE>
__device__ __forceinline__ T m3_ring_r(const M3Ctx<T>& c, int sj, int sp, int sm, int sb, int ro, bool in, int j, T sA,
                                       T& prev) {
    using G = M3<T>;
    const bool out = (unsigned)j >= (unsigned)c.n || !in;
    if (!CACHE && out) return T(0);
    const T b = c.bs[sb * G::BS + ro];
    if constexpr (FZ) {
        return b;
    } else {
        const T* xj = c.xs + sj * G::XS + G::RW + ro;
        const T xp0 = c.xs[sp * G::XS + G::RW + ro];
        T xm0;
        if constexpr (CACHE) {
            xm0 = prev;
            prev = xj[0];
        } else {
            xm0 = c.xs[sm * G::XS + G::RW + ro];
        }
        const T r = residual3d<T>(b, xj[0], xp0, xm0, xj[G::RW], xj[-G::RW], xj[1], xj[-1], sA);
        return (CACHE && out) ? T(0) : r;
    }
}

// tile-local coordinates of ring point i (0 .. NRING-1): consecutive threads take consecutive
// points, so the top/bottom ring rows are read as contiguous shared-memory runs
template <class T>
__device__ __forceinline__ void m3_ring_pt(int i, int& ry, int& rx) {
    using G = M3<T>;
    if (i < G::TX) {
        ry = -1, rx = i;
    } else if (i < 2 * G::TX) {
        ry = G::TY, rx = i - G::TX;
    } else if (i < 2 * G::TX + G::TY) {
        ry = i - 2 * G::TX, rx = -1;
    } else if (i < 2 * G::TX + 2 * G::TY) {
        ry = i - 2 * G::TX - G::TY, rx = G::TX;
    } else {
        const int q = i - 2 * G::TX - 2 * G::TY;
        ry = (q & 2) ? G::TY : -1;
        rx = (q & 1) ? G::TX : -1;
    }
}

template <class T, int S, bool FZ, int NM, int P>
__device__ __forceinline__ void m3_step(const M3Ctx<T>& c, const CUtensorMap* xmap, const CUtensorMap* bmap,
                                        const CUtensorMap* emap, int k, T (&X)[3][2][M3<T>::VEC],
                                        T (&R)[3][2][M3<T>::VEC], T (&XP)[M3<T>::NRP], int& ecs, const Terms<T>& M,
                                        T sA, T sM, T omega, double& nacc) {
    using G = M3<T>;
    using SP = M3S<T, NM>;
    using O = Op<T>;
    constexpr bool PC = SP::PC;
    static_assert(!PC || (S != SHAPE_GENERIC && !FZ), "K3 + K1: named shapes, a given iterate");
    constexpr int VEC = G::VEC;
    constexpr int RW = G::RW;
    // P = k mod 3 fixes the register-array and r / b ring indices at compile time; the x stage
    // slots are runtime (k mod 4), which keeps the unrolled march at 3 steps (a 12-step unroll
    // made every ring index a constant but overflowed the instruction cache in the larger variants)
    static_assert(M3_ST == 4, "stage slots are k & 3");
    const int sj = k & 3, sp = (k + 1) & 3, sm = (k + 3) & 3, s2 = (k + 2) & 3;
    const int bj_slot = PC ? (P + 2) % 3 : sj;  // b(j): K3 + K1 stages b(q0 + 1 + i) in slot i % 3
    constexpr int ic = P % 3, ip = (P + 1) % 3, im = (P + 2) % 3;
    // r ring: planes j, j-1, j-2 (the two-plane ring of the K3 + K1 variant never reads r(j-2))
    constexpr int rj = P % SP::RRD, rj1 = (P + SP::RRD - 1) % SP::RRD, rj2 = (P + 1) % SP::RRD;
    const int j = c.q0 + k;
    // generic shapes read r(j-3)'s ring slot in the previous step's output phase
    // (NM == 3 reads r(j-3)'s slot as r(j-2) in its output phase)
    if constexpr (S == SHAPE_GENERIC || NM == 3) __syncthreads();
    if constexpr (PC) {
        // plane j+1 arrived (and was corrected) a step ago; plane j+2 is corrected in this step
        if (j + 2 <= c.q_last) mbar_wait(&c.full[s2], (uint32_t)(((k + 2) / M3_ST) & 1));
    } else {
        mbar_wait(&c.full[sp], (uint32_t)(((k + 1) / M3_ST) & 1));
    }
    const bool plane_in = (unsigned)j < (unsigned)c.n;

    // ---- r(j) at the two owned rows -------------------------------------------------------
    T* rpl = c.rr + rj * G::RS;
#pragma unroll
    for (int yy = 0; yy < 2; ++yy) {
        const int row = c.yl + yy;
        T bj[VEC];
        V16<T>::ld(c.bs + bj_slot * G::BS + (row + 1) * RW + VEC + c.xl, bj);
        if constexpr (FZ) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) R[ic][yy][v] = bj[v];
        } else {
            const T* xrow = c.xs + sj * G::XS + (row + 2) * RW + VEC + c.xl;
            V16<T>::ld(c.xs + sp * G::XS + (row + 2) * RW + VEC + c.xl, X[ip][yy]);
            T up[VEC], dn[VEC];
            if (yy == 0) {
                V16<T>::ld(xrow - RW, up);
#pragma unroll
                for (int v = 0; v < VEC; ++v) dn[v] = X[ic][1][v];
            } else {
                V16<T>::ld(xrow + RW, dn);
#pragma unroll
                for (int v = 0; v < VEC; ++v) up[v] = X[ic][0][v];
            }
            // horizontal neighbours from the adjacent lanes (a warp spans a whole tile row); only
            // the tile-edge lanes read the staged halo columns
            T left = __shfl_up_sync(0xffffffffu, X[ic][yy][VEC - 1], 1);
            T right = __shfl_down_sync(0xffffffffu, X[ic][yy][0], 1);
            if ((c.tid & 31) == 0) left = xrow[-1];
            if ((c.tid & 31) == 31) right = xrow[VEC];
#pragma unroll
            for (int v = 0; v < VEC; ++v) {
                const T xe = v + 1 < VEC ? X[ic][yy][v + 1] : right;
                const T xw = v > 0 ? X[ic][yy][v - 1] : left;
                R[ic][yy][v] = residual3d<T>(bj[v], X[ic][yy][v], X[ip][yy][v], X[im][yy][v], dn[v], up[v], xe, xw, sA);
            }
        }
        if (!plane_in || c.edge) {
#pragma unroll
            for (int v = 0; v < VEC; ++v)
                if (!plane_in || c.y0 + row >= c.n || c.x0 + c.xl + v >= c.n) R[ic][yy][v] = T(0);
        }
        if ((NM == 1 || NM == 2) && j >= c.z0 && j < c.z_end) {
#pragma unroll
            for (int v = 0; v < VEC; ++v) nacc += (double)R[ic][yy][v] * (double)R[ic][yy][v];
        }
        if (NM != 2) V16<T>::st(rpl + (row + 1) * RW + VEC + c.xl, R[ic][yy]);
    }
    // ---- r(j) on the one-point ring of the tile, spread over all warps ------------------------
    if (NM != 2) {
#pragma unroll
        for (int i = 0; i < G::NRP; ++i) {
            if (c.rro[i] >= 0)
                rpl[c.rro[i]] = m3_ring_r<T, FZ, !FZ>(c, sj, sp, sm, bj_slot, c.rro[i], c.rin[i], j, sA, XP[i]);
        }
    }
    if constexpr (PC) {
        // x + P e on the staged plane j+2 (tile and halo), in place, a step before anything reads
        // it: independent of the r(j) work above, ordered before the next step by the barrier below
        if (j + 2 <= c.q_last) m3_correct_plane<T>(c, j + 2, s2, ecs);
        // ecs follows floor(q/2) mod EST of the plane corrected next
        if (j & 1) ecs = ecs == G::EST - 1 ? 0 : ecs + 1;
    }
    __syncthreads();
    // x(j)'s stage is dead from here on: the step's own reads are done, the ring points' x(j-1)
    // of the next step comes from registers (XP), and the output phase reads r planes and
    // registers only.  It takes plane j+4 (three steps of lead; K3 + K1: two, see M3S).
    if (c.tid == 0 && j + M3_ST <= c.q_last) m3_issue<T, FZ, NM>(c, xmap, bmap, emap, j + M3_ST, sj);
    if constexpr (NM == 3) {
        if ((j & 1) == 0 && j >= c.z0 + 1)
            m3_restrict_out<T>(c, j, c.rr + rj * G::RS, c.rr + rj1 * G::RS, c.rr + rj2 * G::RS, R[ic], R[im], R[ip]);
        return;
    }
    if (NM == 2 || j - 1 < c.z0) return;

    // ---- output plane j-1 -------------------------------------------------------------------
    const T* r1 = c.rr + rj1 * G::RS;  // r(j-1)
    const T* r0 = c.rr + rj * G::RS;   // r(j)
    const T* r2 = c.rr + rj2 * G::RS;  // r(j-2)
    const int nt = tnt<T, S>(M);
#pragma unroll
    for (int yy = 0; yy < 2; ++yy) {
        const int row = c.yl + yy;
        const int so = (row + 1) * RW + VEC + c.xl;  // own position in an r plane
        T out[VEC];
        // r(j-1) one column left of the lane's first / right of its last column: adjacent lanes
        // (the tile-edge lanes read the shared r plane)
        T rl = __shfl_up_sync(0xffffffffu, R[im][yy][VEC - 1], 1);
        T rr = __shfl_down_sync(0xffffffffu, R[im][yy][0], 1);
        if ((c.tid & 31) == 0) rl = r1[so - 1];
        if ((c.tid & 31) == 31) rr = r1[so + VEC];
#pragma unroll
        for (int v = 0; v < VEC; ++v) {
            T acc = T(0);
            if constexpr (S == SHAPE_GENERIC) {
                // runtime term list: every r value (own points included) is in the shared r ring,
                // so a rolled loop keeps the unrolled body small
#pragma unroll 1
                for (int t = 0; t < nt; ++t) {
                    const int o0 = M.off[t][0];
                    const T* pl = o0 == 0 ? r1 : (o0 > 0 ? r0 : r2);
                    acc = O::add(acc, O::mul(M.c[t], pl[so + M.off[t][1] * RW + v + M.off[t][2]]));
                }
            } else {
#pragma unroll
            for (int t = 0; t < ShapeT<(S == SHAPE_GENERIC ? 1 : S)>::nt; ++t) {
                const int o0 = toff<T, S>(M, t, 0), o1 = toff<T, S>(M, t, 1), o2 = toff<T, S>(M, t, 2);
                T val;
                if (o1 == 0 && o2 == 0) {
                    val = o0 == 0 ? R[im][yy][v] : (o0 > 0 ? R[ic][yy][v] : R[ip][yy][v]);
                } else if (o0 == 0 && o2 == 0 && ((o1 > 0 && yy == 0) || (o1 < 0 && yy == 1))) {
                    val = R[im][1 - yy][v];  // in-plane row neighbour held by this thread
                } else if (o0 == 0 && o1 == 0 && v + o2 >= 0 && v + o2 < VEC) {
                    val = R[im][yy][v + o2];
                } else if (o0 == 0 && o1 == 0 && (o2 == -1 || o2 == 1)) {
                    val = o2 < 0 ? rl : rr;
                } else {
                    const T* pl = o0 == 0 ? r1 : (o0 > 0 ? r0 : r2);
                    val = pl[so + o1 * RW + v + o2];
                }
                acc = O::add(acc, O::mul(M.c[t], val));
            }
            }
            out[v] = relax<T>(FZ ? T(0) : X[im][yy][v], acc, sM, omega);
        }
        T* dst = c.obase + (long long)(j - 1) * c.pp + (long long)yy * c.px;
        if (!c.edge) {
            V16<T>::st(dst, out);
        } else if (c.y0 + row < c.n) {
            if (c.x0 + c.xl + VEC <= c.n) {
                V16<T>::st(dst, out);
            } else {
#pragma unroll
                for (int v = 0; v < VEC; ++v)
                    if (c.x0 + c.xl + v < c.n) dst[v] = out[v];
            }
        }
    }
}

template <class T, int S, bool FZ, int NM>
__global__ void __launch_bounds__(M3_THREADS, 2)
    k_sweep3d_march(Layout L, const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap bmap,
                    const __grid_constant__ CUtensorMap emap, const T* __restrict__ x, T* __restrict__ xo, Terms<T> M,
                    T sA, T sM, T omega, int planes, NormOut no, Layout Lc) {
    using G = M3<T>;
    using SP = M3S<T, NM>;
    constexpr int VEC = G::VEC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    M3Ctx<T> c;
    c.xs = reinterpret_cast<T*>(smem_raw);
    c.bs = c.xs + M3_ST * G::XS;
    c.rr = c.bs + SP::BST * G::BS;
    c.es = c.rr + SP::RRD * G::RS;
    c.full = reinterpret_cast<uint64_t*>(c.es + (SP::PC ? G::EST * G::ES : 0));
    c.tid = threadIdx.x;
    c.n = L.n;
    c.px = L.px;
    c.pp = L.pp;
    c.x0 = blockIdx.x * G::TX;
    c.y0 = blockIdx.y * G::TY;
    int z_end;
    if constexpr (NM == 3) {  // chunk = coarse planes [z*planes, (z+1)*planes): fine r planes 2I0 .. 2I1
        c.z0 = 2 * blockIdx.z * planes + 1;
        z_end = min(2 * (blockIdx.z + 1) * planes, 2 * Lc.n);
        c.cb = xo;
        c.cpx = Lc.px;
        c.cpp = Lc.pp;
        c.corg = Lc.origin;
        c.cm = Lc.n;
    } else {
        c.z0 = blockIdx.z * planes;
        z_end = min(c.z0 + planes, c.n);
    }
    c.z_end = z_end;
    c.q0 = c.z0 - 2;
    c.q_last = z_end + 1;
    c.yl = (threadIdx.x >> 5) * 2;
    c.xl = (threadIdx.x & 31) * VEC;
    c.edge = c.x0 + G::TX > c.n || c.y0 + G::TY > c.n;
#pragma unroll
    for (int i = 0; i < G::NRP; ++i) {
        const int p = i * M3_THREADS + (int)threadIdx.x;
        int ry = 0, rx = 0;
        m3_ring_pt<T>(p, ry, rx);
        c.rro[i] = p < G::NRING ? (ry + 1) * G::RW + VEC + rx : -1;
        c.rin[i] = (unsigned)(c.y0 + ry) < (unsigned)c.n && (unsigned)(c.x0 + rx) < (unsigned)c.n;
    }
    c.cx = (int)(L.origin % L.px) + c.x0 - VEC;  // LX + x0 - VEC
    c.ghost = L.ghost;
    c.cy = c.ghost + c.y0 - 2;
    c.obase = xo + L.origin + (long long)(c.y0 + c.yl) * L.px + c.x0 + c.xl;
    if constexpr (SP::PC) {
        c.cm = Lc.n;
        c.eghost = Lc.ghost;
        c.ecx = (int)(Lc.origin % Lc.px) + (c.x0 >> 1) - VEC;
        c.ecy = Lc.ghost + (c.y0 >> 1) - 2;
        c.pc_edge = c.y0 == 0 || c.x0 == 0 || ((c.y0 + G::TY) >> 1) >= Lc.n || ((c.x0 + G::TX + VEC) >> 1) >= Lc.n;
        c.pry[0] = c.yl;
        c.prx[0] = c.xl;
        c.pry[1] = c.prx[1] = 0;
        if (c.tid < G::NHALO) m3_halo_block<T>(c.tid, c.pry[1], c.prx[1]);
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            c.pxo[i] = (c.pry[i] + 2) * G::RW + VEC + c.prx[i];
            // staged coarse tile: row 0 = coarse row y0/2 - 2, column 0 = coarse column x0/2 - VEC
            c.peo[i] = ((c.pry[i] >> 1) + 1) * G::ECW + (c.prx[i] >> 1) + VEC - 1;
        }
    }

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&xmap);
        tma_prefetch_desc(&bmap);
        if (SP::PC) tma_prefetch_desc(&emap);
        for (int i = 0; i < M3_ST; ++i) mbar_init(&c.full[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int q = c.q0; q < c.q0 + M3_ST && q <= c.q_last; ++q)
            m3_issue<T, FZ, NM>(c, &xmap, &bmap, &emap, q, q - c.q0);

    T X[3][2][VEC], R[3][2][VEC];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int yy = 0; yy < 2; ++yy)
#pragma unroll
            for (int v = 0; v < VEC; ++v) X[a][yy][v] = R[a][yy][v] = T(0);
    mbar_wait(&c.full[0], 0);
    mbar_wait(&c.full[1], 0);
    T XP[G::NRP];
#pragma unroll
    for (int i = 0; i < G::NRP; ++i) XP[i] = T(0);
    if constexpr (SP::PC) {  // planes q0 .. q0+2 corrected before the march (then two planes ahead)
        m3_correct_plane<T>(c, c.q0, 0, G::eslot(c.q0 >> 1));
        m3_correct_plane<T>(c, c.q0 + 1, 1, G::eslot((c.q0 + 1) >> 1));
        mbar_wait(&c.full[2], 0);
        m3_correct_plane<T>(c, c.q0 + 2, 2, G::eslot((c.q0 + 2) >> 1));
        __syncthreads();
    }
    if (!FZ) {
        // x(q0) at this thread's ring point(s): x(j-1) of the first step
#pragma unroll
        for (int i = 0; i < G::NRP; ++i)
            if (c.rro[i] >= 0) XP[i] = c.xs[G::RW + c.rro[i]];
#pragma unroll
        for (int yy = 0; yy < 2; ++yy) {
            V16<T>::ld(c.xs + 0 * G::XS + (c.yl + yy + 2) * G::RW + VEC + c.xl, X[0][yy]);
            V16<T>::ld(c.xs + 1 * G::XS + (c.yl + yy + 2) * G::RW + VEC + c.xl, X[1][yy]);
        }
    }
    // every read of plane q0's stage is done (no step reads it: x(q0) lives in registers, b(q0) is
    // unused): it takes plane q0 + 4
    __syncthreads();
    if (threadIdx.x == 0 && c.q0 + M3_ST <= c.q_last) m3_issue<T, FZ, NM>(c, &xmap, &bmap, &emap, c.q0 + M3_ST, 0);
    double nacc = 0.0;
    int ecs = SP::PC ? G::eslot((c.q0 + 3) >> 1) : 0;  // step k = 1 corrects plane q0 + 3
    const int K = z_end - c.q0;  // steps k = 1..K (planes j = z0-1 .. z_end)
    for (int kb = 0; kb <= K; kb += 3) {
#define M3STEP(p)                                                                            \
    if (kb + (p) >= 1 && kb + (p) <= K)                                                     \
        m3_step<T, S, FZ, NM, (p)>(c, &xmap, &bmap, &emap, kb + (p), X, R, XP, ecs, M, sA, sM, omega, nacc);
        M3STEP(0) M3STEP(1) M3STEP(2)
#undef M3STEP
    }
    if (NM == 1 || NM == 2) norm_epilogue(nacc, no);
}

// ------------------------------------------------------------------------------------------
// host side: tensor maps + launch
// ------------------------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 3-D map over a whole padded level allocation (cols, rows, planes), box = (RW, rows, 1)
template <class T>
static cudaError_t make_map(CUtensorMap* map, const Layout& L, const T* base, int box_rows, int box_cols = M3<T>::RW) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {(cuuint64_t)L.px, (cuuint64_t)(L.pp / L.px), (cuuint64_t)(L.alloc / L.pp)};
    const cuuint64_t strides[2] = {(cuuint64_t)L.px * sizeof(T), (cuuint64_t)L.pp * sizeof(T)};
    const cuuint32_t box[3] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                    const_cast<T*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class T, int S, bool FZ, int NM>
cudaError_t launch_sweep3d_march(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA, T sM,
                                 T omega, const NormOut& no, cudaStream_t s, const Layout* Lc, const T* ec) {
    using G = M3<T>;
    constexpr size_t smem = M3S<T, NM>::smem;
    {  // per device, so set on every launch (host-side, cheap)
        cudaError_t e = cudaFuncSetAttribute(k_sweep3d_march<T, S, FZ, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
    }
    // base pointers of the allocations (the layout origin is an offset into them)
    const T* xbase = x ? x : b;  // FZ never reads x; any valid map works
    CUtensorMap xm, bm;
    cudaError_t e = make_map<T>(&xm, L, xbase, G::XR);
    if (e != cudaSuccess) return e;
    e = make_map<T>(&bm, L, b, G::BR);
    if (e != cudaSuccess) return e;
    CUtensorMap em = bm;  // K3 + K1: the coarse correction tile
    if (NM == 4) {
        e = make_map<T>(&em, *Lc, ec, G::ER, G::ECW);
        if (e != cudaSuccess) return e;
    }
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep3d_march<T, S, FZ, NM>, M3_THREADS, smem);
        if (occ <= 0) occ = 1;
    }
    const int tx = (L.n + G::TX - 1) / G::TX, ty = (L.n + G::TY - 1) / G::TY;
    const int slots = num_sms() * occ;
    const int span = NM == 3 ? Lc->n : L.n;  // NM == 3 chunks coarse planes
    int chunks = march_chunks(tx * ty, slots, span, NM == 3 ? 4 : 8, NM == 3 ? 2 : 3);
    const int planes = (span + chunks - 1) / chunks;
    chunks = (span + planes - 1) / planes;
    dim3 g(tx, ty, chunks);
    return launch_k(k_sweep3d_march<T, S, FZ, NM>, g, dim3(M3_THREADS), smem, s, L, xm, bm, em, x, xo, M, sA, sM,
                      omega, planes, no, Lc ? *Lc : L);
}

#define SPAIMG_M3_INST(T, S, FZ, NM)                                                                           \
    template cudaError_t launch_sweep3d_march<T, S, FZ, NM>(const Layout&, const T*, const T*, T*, const Terms<T>&, \
                                                            T, T, T, const NormOut&, cudaStream_t, const Layout*,     \
                                                            const T*);
#define SPAIMG_M3_INST4(T, S) \
    SPAIMG_M3_INST(T, S, false, 0) SPAIMG_M3_INST(T, S, true, 0) SPAIMG_M3_INST(T, S, false, 1) SPAIMG_M3_INST(T, S, true, 1)
SPAIMG_M3_INST4(double, SHAPE_GENERIC)
SPAIMG_M3_INST4(double, SHAPE_C1)
SPAIMG_M3_INST4(double, SHAPE_STAR7)
SPAIMG_M3_INST4(float, SHAPE_GENERIC)
SPAIMG_M3_INST4(float, SHAPE_C1)
SPAIMG_M3_INST4(float, SHAPE_STAR7)
SPAIMG_M3_INST(double, SHAPE_C1, false, 2)
SPAIMG_M3_INST(float, SHAPE_C1, false, 2)
SPAIMG_M3_INST(double, SHAPE_C1, false, 3)
SPAIMG_M3_INST(float, SHAPE_C1, false, 3)
SPAIMG_M3_INST(double, SHAPE_C1, false, 4)
SPAIMG_M3_INST(float, SHAPE_C1, false, 4)
SPAIMG_M3_INST(double, SHAPE_STAR7, false, 4)
SPAIMG_M3_INST(float, SHAPE_STAR7, false, 4)

}  // namespace spaimg
