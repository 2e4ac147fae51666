// K2: fused residual + full-weighting restriction, rc = restrict(b - A x)
// (reference multigrid.py:176-177 with restrict from :104-119).
//
// 2D: a CTA owns a strip of CW coarse columns (2CW+1 fine columns) and marches down the fine
// rows.  A producer warp streams (x row, b row) pairs with 1-D bulk copies into a ring of
// shared-memory stages; each consumer lane owns one coarse column = two fine columns, keeps
// x(f-1..f+1) and r(f-2..f) of them in registers, and on every even fine row f = 2I+2 forms
// the axis-0 weights t = (0.25 r(2I) + 0.5 r(2I+1)) + 0.25 r(2I+2) and then the axis-1
// weights from its own two t values plus the right neighbour's first one (shuffle / edge
// slot / producer-computed halo column).  HBM traffic: x + b + coarse = 18 B per fine point
// (fp64); r never leaves registers.
#include <cstdlib>

#include "kernels.h"
#include "march.cuh"
#include "ptx.cuh"

namespace spaimg {

constexpr int R2_NW = 4;  // consumer warps
constexpr int R2_ST = 6;  // stage ring depth (= unroll factor)

template <class T> struct R2 {
    static constexpr int V = 16 / (int)sizeof(T);  // 16-byte halo granule
    static constexpr int CW = 32 * R2_NW;          // coarse columns per strip
    static constexpr int RW = 2 * CW + 2 * V;      // staged fine row: [2J0 - V, 2J0 + 2CW + V)
    static constexpr size_t smem = (size_t)2 * R2_ST * RW * sizeof(T) + (R2_NW + 1) * sizeof(T) + 16 + R2_ST * 8;
};

template <class T>
struct R2Ctx {
    T* xs;
    T* bs;
    T* te;  // t edge slots [NW+1]
    uint64_t* full;
    const T* xrow0;
    const T* brow0;
    T* crow0;  // coarse row 0 at own column
    long long px, cpx;
    int sidx, q0, q_last, lane, warp, I0, m, J;
    bool producer;
};

template <class T>
__device__ __forceinline__ void r2_issue(const R2Ctx<T>& c, int q, int slot) {
    constexpr int RW = R2<T>::RW;
    constexpr uint32_t rb = RW * sizeof(T);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&c.full[slot], 2 * rb);
    bulk_g2s(c.xs + slot * RW, c.xrow0 + (long long)q * c.px, rb, &c.full[slot]);
    bulk_g2s(c.bs + slot * RW, c.brow0 + (long long)q * c.px, rb, &c.full[slot]);
}

template <class T, int P>
__device__ __forceinline__ void r2_step(const R2Ctx<T>& c, int k, T (&X)[3][2], T (&R)[3][2], T (&RH)[3], T sA) {
    constexpr int RW = R2<T>::RW;
    constexpr int CW = R2<T>::CW;
    constexpr int V = R2<T>::V;
    constexpr int sf = P % R2_ST, sp = (P + 1) % R2_ST, sm = (P + R2_ST - 1) % R2_ST;  // rows f, f+1, f-1
    constexpr int ic = P % 3, ip = (P + 1) % 3, im = (P + 2) % 3;
    constexpr bool out_step = (P % 2) == 1;  // f = q0 + k even  <=>  k odd (q0 is odd)
    const int f = c.q0 + k;
    mbar_wait(&c.full[sp], (uint32_t)(((k + 1) / R2_ST) & 1));
    T t[2];
    if (!c.producer) {
        T bf[2];
        V16<T>::ld2(c.bs + sf * RW + c.sidx, bf);
        V16<T>::ld2(c.xs + sp * RW + c.sidx, X[ip]);
        const T left = c.xs[sf * RW + c.sidx - 1];
        const T right = c.xs[sf * RW + c.sidx + 2];
        R[ic][0] = residual2d<T>(bf[0], X[ic][0], X[ip][0], X[im][0], X[ic][1], left, sA);
        R[ic][1] = residual2d<T>(bf[1], X[ic][1], X[ip][1], X[im][1], right, X[ic][0], sA);
        if (out_step && k >= 3) {
            t[0] = fw<T>(R[ip][0], R[im][0], R[ic][0]);  // rows f-2, f-1, f
            t[1] = fw<T>(R[ip][1], R[im][1], R[ic][1]);
            if (c.lane == 0) c.te[c.warp] = t[0];
        }
    } else if (c.lane == 0) {
        // halo fine column 2J0 + 2CW
        const int si = V + 2 * CW;
        RH[ic] = residual2d<T>(c.bs[sf * RW + si], c.xs[sf * RW + si], c.xs[sp * RW + si], c.xs[sm * RW + si],
                               c.xs[sf * RW + si + 1], c.xs[sf * RW + si - 1], sA);
        if (out_step && k >= 3) c.te[R2_NW] = fw<T>(RH[ip], RH[im], RH[ic]);
    }
    named_bar_sync(1, (R2_NW + 1) * 32);
    if (c.producer) {
        if (c.lane == 0 && f - 1 + R2_ST <= c.q_last) r2_issue<T>(c, f - 1 + R2_ST, sm);
        return;
    }
    if (out_step && k >= 3) {
        T tn = __shfl_down_sync(0xffffffffu, t[0], 1);
        if (c.lane == 31) tn = c.te[c.warp + 1];
        const int I = f / 2 - 1;
        if (c.J < c.m) c.crow0[(long long)I * c.cpx] = fw<T>(t[0], t[1], tn);
    }
}

template <class T>
__global__ void __launch_bounds__((R2_NW + 1) * 32) k_residual_restrict2d(Layout Lf, Layout Lc, const T* __restrict__ x,
                                                                           const T* __restrict__ b, T* __restrict__ bc,
                                                                           T sA, int rows) {
    constexpr int RW = R2<T>::RW;
    constexpr int V = R2<T>::V;
    constexpr int CW = R2<T>::CW;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    R2Ctx<T> c;
    c.xs = reinterpret_cast<T*>(smem_raw);
    c.bs = c.xs + R2_ST * RW;
    c.te = c.bs + R2_ST * RW;
    c.full = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(c.te + R2_NW + 1) + 15) & ~uintptr_t(15));
    c.warp = threadIdx.x >> 5;
    c.lane = threadIdx.x & 31;
    c.producer = c.warp == R2_NW;
    c.m = Lc.n;
    const int J0 = blockIdx.x * CW;
    c.I0 = blockIdx.y * rows;
    const int I_end = min(c.I0 + rows, c.m);
    c.q0 = 2 * c.I0 - 1;      // first staged fine row
    c.q_last = 2 * I_end + 1;  // last staged fine row
    c.px = Lf.px;
    c.cpx = Lc.px;
    const int lc = (c.producer ? 0 : c.warp) * 32 + c.lane;  // coarse column within the strip
    c.J = J0 + lc;
    c.sidx = V + 2 * lc;
    c.xrow0 = x + Lf.origin + (2 * J0 - V);
    c.brow0 = b + Lf.origin + (2 * J0 - V);
    c.crow0 = bc + Lc.origin + c.J;

    if (threadIdx.x == 0) {
        for (int i = 0; i < R2_ST; ++i) mbar_init(&c.full[i], 1);
        mbar_fence_init();
    }
    __syncthreads();
    if (c.producer && c.lane == 0)
        for (int q = c.q0; q < c.q0 + R2_ST && q <= c.q_last; ++q) r2_issue<T>(c, q, q - c.q0);

    T X[3][2], R[3][2], RH[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        RH[a] = T(0);
        X[a][0] = X[a][1] = R[a][0] = R[a][1] = T(0);
    }
    mbar_wait(&c.full[0], 0);
    mbar_wait(&c.full[1], 0);
    if (!c.producer) {
        V16<T>::ld2(c.xs + 0 * RW + c.sidx, X[0]);
        V16<T>::ld2(c.xs + 1 * RW + c.sidx, X[1]);
    }
    const int K = 2 * I_end - c.q0;  // steps k = 1..K (fine rows 2I0 .. 2I_end)
    for (int kb = 0; kb <= K; kb += R2_ST) {
        if (kb >= 1) r2_step<T, 0>(c, kb, X, R, RH, sA);
        if (kb + 1 <= K) r2_step<T, 1>(c, kb + 1, X, R, RH, sA);
        if (kb + 2 <= K) r2_step<T, 2>(c, kb + 2, X, R, RH, sA);
        if (kb + 3 <= K) r2_step<T, 3>(c, kb + 3, X, R, RH, sA);
        if (kb + 4 <= K) r2_step<T, 4>(c, kb + 4, X, R, RH, sA);
        if (kb + 5 <= K) r2_step<T, 5>(c, kb + 5, X, R, RH, sA);
    }
}

template <class T>
cudaError_t launch_residual_restrict2d_march(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T sA,
                                             cudaStream_t s) {
    constexpr size_t smem = R2<T>::smem;
    constexpr int threads = (R2_NW + 1) * 32;
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_residual_restrict2d<T>, threads, smem);
        if (occ <= 0) occ = 1;
    }
    const int m = Lc.n;
    const int strips = (m + R2<T>::CW - 1) / R2<T>::CW;
    const int slots = num_sms() * occ;
    int chunks = march_chunks(strips, slots, m, 8, 1);
    const int rows = (m + chunks - 1) / chunks;
    chunks = (m + rows - 1) / rows;
    dim3 g(strips, chunks);
    return launch_k(k_residual_restrict2d<T>, g, dim3(threads), smem, s, Lf, Lc, x, b, bc, sA, rows);
}

template cudaError_t launch_residual_restrict2d_march<double>(const Layout&, const Layout&, const double*,
                                                              const double*, double*, double, cudaStream_t);
template cudaError_t launch_residual_restrict2d_march<float>(const Layout&, const Layout&, const float*, const float*,
                                                             float*, float, cudaStream_t);

}  // namespace spaimg
