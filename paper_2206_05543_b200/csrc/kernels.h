// Host-side launcher declarations for the spaimg sm_100a kernels (internal to the library).
#pragma once

#include <cuda_runtime.h>

#include "spaimg_common.cuh"

namespace spaimg {

// typed kernel launch (arguments converted to the kernel's parameter types)
template <class... KP, class... A>
inline cudaError_t launch_k(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.numAttrs = 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KP>(args)...);
}

Layout make_layout(int dim, int N, int esize, int ghost = kGhost);
// checked build only: NaN interior and slack, zero two-cell frame (see spaimg_common.cuh)
template <class T> cudaError_t launch_poison_level(const Layout& L, T* p, cudaStream_t s);

// dense (n^dim, C order) <-> padded interior
template <class T> cudaError_t launch_pad(const Layout& L, const T* dense, T* padded, cudaStream_t s);
template <class T> cudaError_t launch_unpad(const Layout& L, const T* padded, T* dense, cudaStream_t s);

// K0: zero-extended stencil product on dense arrays (any offset radius), stencils.py:136-153
template <class T>
cudaError_t launch_apply_dense(int dim, int N, const T* x, T* out, const Terms<T>& terms, T scale,
                               cudaStream_t s);

// unfused building blocks on padded levels
template <class T>
cudaError_t launch_residual(const Layout& L, const T* x, const T* b, T* r, T sA, cudaStream_t s);
template <class T>
cudaError_t launch_relax(const Layout& L, const T* x, const T* r, T* xo, const Terms<T>& M, int shape, T sM,
                         T omega, cudaStream_t s);
template <class T>
cudaError_t launch_restrict(const Layout& Lf, const Layout& Lc, const T* r, T* bc, cudaStream_t s);

// K1: fused smoothing sweep x' = x + omega M (b - A x); from_zero => x == 0 (x not read)
// no != nullptr additionally appends ||b - A x|| (of the INPUT x) to the device history.
template <class T>
cudaError_t launch_sweep(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, int shape, T sA,
                         T sM, T omega, bool from_zero, cudaStream_t s, const NormOut* no = nullptr);
bool sweep_fused_supported(int dim, int shape);
// K3 + K1: xo = sweep(x + P e) (prolongation + correction fused into the first post-sweep)
bool sweep_pc_supported(const Layout& L, int shape);
// two smoothing steps in one 2D march (second sweep pipelined three rows behind the first):
// xo = sweep(sweep(x)) [from_zero: x == 0; no: the input residual's norm], and the K3 variant
// xo = sweep(sweep(x + P e)); 2D marching levels, named shapes
bool sweep2_supported(const Layout& L, int shape);
template <class T>
cudaError_t launch_sweep2(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, int shape, T sA, T sM,
                          T omega, bool from_zero, cudaStream_t s, const NormOut* no = nullptr);
template <class T>
cudaError_t launch_sweep2_pc(const Layout& L, const Layout& Lc, const T* x, const T* e, const T* b, T* xo,
                             const Terms<T>& M, int shape, T sA, T sM, T omega, cudaStream_t s);
template <class T>
cudaError_t launch_sweep_pc(const Layout& L, const Layout& Lc, const T* x, const T* e, const T* b, T* xo,
                            const Terms<T>& M, int shape, T sA, T sM, T omega, cudaStream_t s);
// K4 through the marching kernels: ||b - A x|| appended to the device history
template <class T>
cudaError_t launch_norm_march(const Layout& L, const T* x, const T* b, T sA, const NormOut& no, cudaStream_t s);

// K2: fused residual + full-weighting restriction
template <class T>
cudaError_t launch_residual_restrict(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T sA,
                                     cudaStream_t s);
// K2 / K1 for small levels: flat one-wave kernels (kernels_flat.cu); levels with mesh count
// N <= flat_threshold(dim) use them instead of the marching kernels
int flat_threshold(int dim);
// K2 fused with the coarse level's first (zero-start) pre-sweep: bc = restrict(b - A x),
// xc = 0 + omega (M bc) sMc  (radius-1 M; small levels)
template <class T>
cudaError_t launch_residual_restrict_fz(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T* xc,
                                        const Terms<T>& M, int shape, T sA, T sMc, T omega, cudaStream_t s);
template <class T>
cudaError_t launch_residual_restrict_flat(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T sA,
                                          cudaStream_t s);

// K3: fused prolongation + correction xo = xi + P e (xi == xo allowed); acc=false stores P e alone
template <class T>
cudaError_t launch_prolong_correct(const Layout& Lf, const Layout& Lc, const T* xi, T* xo, const T* e, cudaStream_t s,
                                   bool acc = true);

// K4: deterministic two-stage ||b - A x||_2 into norms[slot] (double); partials/counter scratch
constexpr int kNormBlocks = 592;  // 4 x 148 SMs
template <class T>
cudaError_t launch_residual_norm(const Layout& L, const T* x, const T* b, T sA, double* partials,
                                 unsigned* counter, double* norms, int slot, int* slot_dev, cudaStream_t s);

// K5: coarse direct solve (LAPACK getrs order, Appendix A.5/A.6)
template <class T>
cudaError_t launch_coarse_solve(const Layout& L, const T* b, T* x, const T* lu, const int* piv, int nlu,
                                cudaStream_t s);

// numpy Generator(PCG64).uniform(low, high) draws in C order on the device, bitwise
// (kernels_rng.cu); st = {state_hi, state_lo, inc_hi, inc_lo} of the seeded generator
template <class T>
cudaError_t launch_fill_uniform(T* out, long long count, const unsigned long long st[4], double low, double high,
                                cudaStream_t s);

// K5+: the shared-memory coarse-grid engine (kernels_tail.cu).  Every level from a size
// threshold down lives in one CTA's shared memory; the CTA interprets the host-recorded op list
// of the V/W recursion below its entry level (multigrid.py:157-185), each op point-parallel
// over the op's level, ops separated by barriers over the warps involved.
constexpr int kTailThreads = 512;
enum TailOpType : int {
    TAIL_RES = 0,      // r = b - A x                               (multigrid.py:99, :176)
    TAIL_RELAX = 1,    // x = x + omega ((M r) sM), in place         (multigrid.py:100)
    TAIL_RELAX0 = 2,   // x = 0 + omega ((M b) sM): first sweep from a zero iterate (r == b)
    TAIL_ZERO = 3,     // x = 0 (nu1 == 0 on a zero start)
    TAIL_FW = 4,       // coarse b = full weighting of r             (multigrid.py:104-119)
    TAIL_PROLONG = 5,  // x = x + P (coarse x)                       (multigrid.py:122-144, :184)
    TAIL_COARSE = 6,   // x = (LU)^-1 b in getrs order                (multigrid.py:147-154)
    // fused ops of the compile-time engine (kernels_tail_fast.cuh; host-side labels only)
    TAIL_RESFW = 7,        // RES + FW
};
// One op = one packed word (host-recorded): type | level << 3 | nw << 6 | bw << 11 | bid << 16
//   level: index into TailArgs::lv (0 = the entry level); FW / PROLONG also use level + 1
//   nw:    warps executing the op (a prefix of the CTA)
//   bw:    warps meeting at the barrier before the op: max(nw of this op and of the previous one)
//   bid:   barrier for bw warps: 0 = __syncthreads, kTailSyncWarp = __syncwarp, else a named id
constexpr int kTailMaxOps = 1536;
constexpr int kTailMaxLevels = 8;
constexpr int kTailMaxLU = 27;   // coarse systems up to 27 unknowns keep their factors in the parameters
constexpr int kTailSyncWarp = 31;
__host__ __device__ constexpr unsigned tail_op_word(int type, int level, int nw, int bw, int bid) {
    return (unsigned)type | (unsigned)level << 3 | (unsigned)nw << 6 | (unsigned)bw << 11 | (unsigned)bid << 16;
}
// a level in the engine's shared memory: array offsets are element offsets, from the start of the
// level-array block, of each array's interior point 0
template <class T> struct TailLv {
    int n;        // interior points per axis
    int logw;     // the level's points are mapped onto a W^dim box, W = 1 << logw
    int s0, s1;   // element pitch of axis 0 and (3D) axis 1
    int x, b, r;  // arrays (r = -1 on the coarse level)
    int pad;
    T sA, sM;
};
// Everything the engine reads per op lives in the kernel parameters (constant bank): the op
// words, the level table and the coarse LU factors, so an op costs no shared-memory fetch and
// the substitution's coefficients are DFMA constant operands.
template <class T> struct TailArgs {
    int nops, nlv, nlu;
    int gamma, nu1, nu2;     // the cycle (the compile-time engine walks the recursion itself)
    int entry_fz;            // the entry level starts from a zero iterate
    int fast_le, fast_lc;    // > 0: the compile-time engine for entry / coarse levels of n = 2^le - 1 / 2^lc - 1
    int arr_elems;           // T elements of the level-array block
    int zero_from;           // elements [zero_from, arr_elems) are zeroed on entry (level 0's r onwards)
    int frame;               // F: zero frame width of the shared-memory arrays (stencil radius)
    size_t smem;             // dynamic shared memory bytes (the level arrays [+ the LU work vector])
    Terms<T> M;
    T omega;
    // the entry level: b and the start iterate come from its global buffers (zero frames
    // included), the result goes back to gx (in place)
    Layout gL;
    const T* gb;
    T* gx;
    int shape;               // SHAPE_* of M: named shapes get compile-time stencil offsets
    long long* prof;         // diagnostics (SPAIMG_TAIL_PROF=1): clock64() at the start of each op
    // coarse factors for nlu > kTailMaxLU (global memory; copied to shared memory on entry)
    const T* coarse_g;       // [nlu*nlu: -LU off the diagonal, row-major | U_jj | 1/U_jj]
    const int* coarse_idx_g; // [b offsets of the permuted rows | x offsets]
    TailLv<T> lv[kTailMaxLevels];
    // coarse factors for nlu <= kTailMaxLU: row-major -LU off the diagonal, U_jj, 1/U_jj, and the
    // b offsets of the permuted rows / x offsets of the unknowns (getrs row interchanges folded in)
    T lu[kTailMaxLU * kTailMaxLU];
    T dg[kTailMaxLU], rc[kTailMaxLU];
    int cin[kTailMaxLU], cout[kTailMaxLU];
    unsigned ops[kTailMaxOps];
};
template <class T> cudaError_t launch_tail(const TailArgs<T>& a, cudaStream_t s);
// the compile-time engine (kernels_tail_fast{2,3}d.cu): which entry / coarse sizes and shapes it
// is instantiated for; cudaErrorNotSupported otherwise
constexpr int kTailFastLE2 = 6, kTailFastLE3 = 4;
inline bool tail_fast_shape(int dim, int shape) {
    return dim == 2 ? (shape == SHAPE_C1 || shape == SHAPE_STAR5 || shape == SHAPE_BOX9)
                    : (shape == SHAPE_C1 || shape == SHAPE_STAR7);
}
template <class T> cudaError_t launch_tail_fast2d(const TailArgs<T>& a, cudaStream_t s);
template <class T> cudaError_t launch_tail_fast3d(const TailArgs<T>& a, cudaStream_t s);

}  // namespace spaimg
