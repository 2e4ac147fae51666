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
// tile: 2(TX+TY)/(TX*TY) extra).  The step loop is unrolled by 12 = lcm(4 stages, 3 rows) so
// every ring index is a compile-time constant.
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
    static constexpr size_t smem = (size_t)(M3_ST * (XS + BS) + M3_RR * RS) * sizeof(T) + M3_ST * 8;
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
    int cx, cy;  // TMA coordinates of the tile's stage origin (x stage)
    int ghost;   // the layout's ghost planes/rows (TMA coordinate of interior 0)
    // NM == 3 (K2 residual + restriction): coarse output level
    T* cb;
    long long cpx, cpp, corg;
    int cm;
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

template <class T, bool FZ>
__device__ __forceinline__ void m3_issue(const M3Ctx<T>& c, const CUtensorMap* xm, const CUtensorMap* bm, int q,
                                         int slot) {
    using G = M3<T>;
    constexpr uint32_t xb = G::XR * G::RW * sizeof(T), bb = G::BR * G::RW * sizeof(T);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&c.full[slot], FZ ? bb : xb + bb);
    if (!FZ) tma_load_3d(c.xs + slot * G::XS, xm, c.cx, c.cy, c.ghost + q, &c.full[slot]);
    tma_load_3d(c.bs + slot * G::BS, bm, c.cx, c.cy + 1, c.ghost + q, &c.full[slot]);
}

// r at a tile-local ring point (ry, rx) of plane j, all operands from shared memory
template <class T, bool FZ>
__device__ __forceinline__ T m3_ring_r(const M3Ctx<T>& c, int sj, int sp, int sm, int ry, int rx, int j, T sA) {
    using G = M3<T>;
    const int gy = c.y0 + ry, gx = c.x0 + rx;
    if ((unsigned)j >= (unsigned)c.n || (unsigned)gy >= (unsigned)c.n || (unsigned)gx >= (unsigned)c.n) return T(0);
    const T b = c.bs[sj * G::BS + (ry + 1) * G::RW + G::VEC + rx];
    if constexpr (FZ) {
        return b;
    } else {
        const T* xj = c.xs + sj * G::XS + (ry + 2) * G::RW + G::VEC + rx;
        const T xp0 = c.xs[sp * G::XS + (ry + 2) * G::RW + G::VEC + rx];
        const T xm0 = c.xs[sm * G::XS + (ry + 2) * G::RW + G::VEC + rx];
        return residual3d<T>(b, xj[0], xp0, xm0, xj[G::RW], xj[-G::RW], xj[1], xj[-1], sA);
    }
}

template <class T, int S, bool FZ, int NM, int P>
__device__ __forceinline__ void m3_step(const M3Ctx<T>& c, const CUtensorMap* xmap, const CUtensorMap* bmap, int k,
                                        T (&X)[3][2][M3<T>::VEC], T (&R)[3][2][M3<T>::VEC], const Terms<T>& M,
                                        T sA, T sM, T omega, double& nacc) {
    using G = M3<T>;
    using O = Op<T>;
    constexpr int VEC = G::VEC;
    constexpr int RW = G::RW;
    constexpr int sj = P % M3_ST, sp = (P + 1) % M3_ST, sm = (P + M3_ST - 1) % M3_ST;
    constexpr int ic = P % 3, ip = (P + 1) % 3, im = (P + 2) % 3;
    constexpr int rj = P % M3_RR, rj1 = (P + 2) % M3_RR, rj2 = (P + 1) % M3_RR;  // r ring: planes j, j-1, j-2
    const int j = c.q0 + k;
    // generic shapes read r(j-3)'s ring slot in the previous step's output phase
    // (NM == 3 reads r(j-3)'s slot as r(j-2) in its output phase)
    if constexpr (S == SHAPE_GENERIC || NM == 3) __syncthreads();
    mbar_wait(&c.full[sp], (uint32_t)(((k + 1) / M3_ST) & 1));
    const bool plane_in = (unsigned)j < (unsigned)c.n;

    // ---- r(j) at the two owned rows -------------------------------------------------------
    T* rpl = c.rr + rj * G::RS;
#pragma unroll
    for (int yy = 0; yy < 2; ++yy) {
        const int row = c.yl + yy;
        T bj[VEC];
        V16<T>::ld(c.bs + sj * G::BS + (row + 1) * RW + VEC + c.xl, bj);
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
        // consecutive threads take consecutive ring points, so the top/bottom ring rows are read
        // as contiguous shared-memory runs
#pragma unroll
        for (int base = 0; base < G::NRING; base += M3_THREADS) {
            const int i = base + c.tid;
            if (i < G::NRING) {
                int ry, rx;
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
                rpl[(ry + 1) * RW + VEC + rx] = m3_ring_r<T, FZ>(c, sj, sp, sm, ry, rx, j, sA);
            }
        }
    }
    __syncthreads();
    if (c.tid == 0 && j - 1 + M3_ST <= c.q_last) m3_issue<T, FZ>(c, xmap, bmap, j - 1 + M3_ST, sm);
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
                // so a rolled loop keeps the 12-step unrolled body small
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
                    const T* __restrict__ x, T* __restrict__ xo, Terms<T> M, T sA, T sM, T omega, int planes,
                    NormOut no, Layout Lc) {
    using G = M3<T>;
    constexpr int VEC = G::VEC;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    M3Ctx<T> c;
    c.xs = reinterpret_cast<T*>(smem_raw);
    c.bs = c.xs + M3_ST * G::XS;
    c.rr = c.bs + M3_ST * G::BS;
    c.full = reinterpret_cast<uint64_t*>(c.rr + M3_RR * G::RS);
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
    c.cx = (int)(L.origin % L.px) + c.x0 - VEC;  // LX + x0 - VEC
    c.ghost = L.ghost;
    c.cy = c.ghost + c.y0 - 2;
    c.obase = xo + L.origin + (long long)(c.y0 + c.yl) * L.px + c.x0 + c.xl;

    if (threadIdx.x == 0) {
        tma_prefetch_desc(&xmap);
        tma_prefetch_desc(&bmap);
        for (int i = 0; i < M3_ST; ++i) mbar_init(&c.full[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (threadIdx.x == 0)
        for (int q = c.q0; q < c.q0 + M3_ST && q <= c.q_last; ++q) m3_issue<T, FZ>(c, &xmap, &bmap, q, q - c.q0);

    T X[3][2][VEC], R[3][2][VEC];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int yy = 0; yy < 2; ++yy)
#pragma unroll
            for (int v = 0; v < VEC; ++v) X[a][yy][v] = R[a][yy][v] = T(0);
    mbar_wait(&c.full[0], 0);
    mbar_wait(&c.full[1], 0);
    if (!FZ) {
#pragma unroll
        for (int yy = 0; yy < 2; ++yy) {
            V16<T>::ld(c.xs + 0 * G::XS + (c.yl + yy + 2) * G::RW + VEC + c.xl, X[0][yy]);
            V16<T>::ld(c.xs + 1 * G::XS + (c.yl + yy + 2) * G::RW + VEC + c.xl, X[1][yy]);
        }
    }
    double nacc = 0.0;
    const int K = z_end - c.q0;  // steps k = 1..K (planes j = z0-1 .. z_end)
    for (int kb = 0; kb <= K; kb += 12) {
#define M3STEP(p)                                                                            \
    if (kb + (p) >= 1 && kb + (p) <= K)                                                     \
        m3_step<T, S, FZ, NM, (p)>(c, &xmap, &bmap, kb + (p), X, R, M, sA, sM, omega, nacc);
        M3STEP(0) M3STEP(1) M3STEP(2) M3STEP(3) M3STEP(4) M3STEP(5)
        M3STEP(6) M3STEP(7) M3STEP(8) M3STEP(9) M3STEP(10) M3STEP(11)
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
static cudaError_t make_map(CUtensorMap* map, const Layout& L, const T* base, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[3] = {(cuuint64_t)L.px, (cuuint64_t)(L.pp / L.px), (cuuint64_t)(L.alloc / L.pp)};
    const cuuint64_t strides[2] = {(cuuint64_t)L.px * sizeof(T), (cuuint64_t)L.pp * sizeof(T)};
    const cuuint32_t box[3] = {(cuuint32_t)M3<T>::RW, (cuuint32_t)box_rows, 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = fn(map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3,
                    const_cast<T*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <class T, int S, bool FZ, int NM>
cudaError_t launch_sweep3d_march(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA, T sM,
                                 T omega, const NormOut& no, cudaStream_t s, const Layout* Lc) {
    using G = M3<T>;
    {  // per device, so set on every launch (host-side, cheap)
        cudaError_t e = cudaFuncSetAttribute(k_sweep3d_march<T, S, FZ, NM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)G::smem);
        if (e != cudaSuccess) return e;
    }
    // base pointers of the allocations (the layout origin is an offset into them)
    const T* xbase = x ? x : b;  // FZ never reads x; any valid map works
    CUtensorMap xm, bm;
    cudaError_t e = make_map<T>(&xm, L, xbase, G::XR);
    if (e != cudaSuccess) return e;
    e = make_map<T>(&bm, L, b, G::BR);
    if (e != cudaSuccess) return e;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_sweep3d_march<T, S, FZ, NM>, M3_THREADS, G::smem);
        if (occ <= 0) occ = 1;
    }
    const int tx = (L.n + G::TX - 1) / G::TX, ty = (L.n + G::TY - 1) / G::TY;
    const int slots = num_sms() * occ;
    const int span = NM == 3 ? Lc->n : L.n;  // NM == 3 chunks coarse planes
    int chunks = march_chunks(tx * ty, slots, span, NM == 3 ? 4 : 8, NM == 3 ? 2 : 3);
    const int planes = (span + chunks - 1) / chunks;
    chunks = (span + planes - 1) / planes;
    dim3 g(tx, ty, chunks);
    return launch_k(k_sweep3d_march<T, S, FZ, NM>, g, dim3(M3_THREADS), G::smem, s, L, xm, bm, x, xo, M, sA, sM,
                      omega, planes, no, Lc ? *Lc : L);
}

#define SPAIMG_M3_INST(T, S, FZ, NM)                                                                           \
    template cudaError_t launch_sweep3d_march<T, S, FZ, NM>(const Layout&, const T*, const T*, T*, const Terms<T>&, \
                                                            T, T, T, const NormOut&, cudaStream_t, const Layout*);
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

}  // namespace spaimg
