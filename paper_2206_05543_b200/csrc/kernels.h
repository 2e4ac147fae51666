// Host-side launcher declarations for the spaimg sm_100a kernels (internal to the library).
#pragma once

#include <cuda_runtime.h>

#include "spaimg_common.cuh"

namespace spaimg {

// launch with the Programmatic-Dependent-Launch attribute when SPAIMG_PDL=1; the kernel
// must call pdl_wait() before its first global memory access
bool pdl_enabled();
template <class... KP, class... A>
inline cudaError_t launch_pdl(void (*k)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, k, static_cast<KP>(args)...);
}

Layout make_layout(int dim, int N, int esize);

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
// K1 + K2: xo = sweep(x) and bc = restrict(b - A xo) in one march (2D marching levels);
// from_zero: x == 0; no != nullptr: the norm of the input residual is appended as well
bool sweep_rr_supported(const Layout& L);
template <class T>
cudaError_t launch_sweep_rr(const Layout& L, const Layout& Lc, const T* x, const T* b, T* xo, T* bc, const Terms<T>& M,
                            int shape, T sA, T sM, T omega, bool from_zero, cudaStream_t s, const NormOut* no);
// K3 + K1: xo = sweep(x + P e) (prolongation + correction fused into the first post-sweep)
bool sweep_pc_supported(const Layout& L);
template <class T>
cudaError_t launch_sweep_pc(const Layout& L, const Layout& Lc, const T* x, const T* e, const T* b, T* xo,
                            const Terms<T>& M, int shape, T sA, T sM, T omega, cudaStream_t s);
bool sweep_norm_supported();
// K4 through the marching kernels: ||b - A x|| appended to the device history
template <class T>
cudaError_t launch_norm_march(const Layout& L, const T* x, const T* b, T sA, const NormOut& no, cudaStream_t s);

// K2: fused residual + full-weighting restriction
template <class T>
cudaError_t launch_residual_restrict(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T sA,
                                     T* scratch_r, cudaStream_t s);
// K2 / K1 for small levels: flat one-wave kernels (kernels_flat.cu); levels with mesh count
// N <= flat_threshold(dim) use them instead of the marching kernels
int flat_threshold(int dim);
// K2 fused with the coarse level's first (zero-start) pre-sweep: bc = restrict(b - A x),
// xc = 0 + omega (M bc) sMc  (radius-1 M; small levels)
template <class T>
cudaError_t launch_residual_restrict_fz(const Layout& Lf, const Layout& Lc, const T* x, const T* b, T* bc, T* xc,
                                        const Terms<T>& M, int shape, T sA, T sMc, T omega, cudaStream_t s);
template <class T>
cudaError_t launch_sweep_pc_flat(const Layout& L, const Layout& Lc, const T* x, const T* e, const T* b, T* xo,
                                 const Terms<T>& M, int shape, T sA, T sM, T omega, cudaStream_t s);
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

// K5+: single-block, shared-memory-resident tail of the cycle (kernels_tail.cu): every level
// from a threshold down runs inside one CTA, interpreting the host-recorded op list of the
// recursion (levels relative to the entry level 0).
enum TailOpType { TAIL_SWEEP = 0, TAIL_ZERO = 1, TAIL_RESTRICT = 2, TAIL_PROLONG = 3, TAIL_COARSE = 4, TAIL_SOLO = 5 };
struct TailOp {
    int type;
    int level;        // index into the tail levels (0 = entry level)
    int a_in, a_out;  // x buffer indices of the level
    int c;            // PROLONG: x buffer of the coarse level holding the correction
    int fz;           // SWEEP: the input iterate is zero (x not read)
    int nthr;         // participating threads (a multiple of 32): the op's largest point count
    int npre;         // threads meeting at the barrier before the op: max(nthr, previous op's nthr)
    int bid_pre, bid_in;  // named-barrier ids for npre / nthr threads (0 = __syncthreads)
};
template <class T> struct TailLevel {
    Layout L;   // compact shared-memory layout (frame = stencil radius)
    T* x[2];    // host side: element offsets into the shared array block
    T* b;
    T* r;
    T sA, sM;
};
template <class T> struct TailArgs {
    const TailLevel<T>* lv;  // device array, nlv entries
    const TailOp* ops;       // device array, nops entries
    int nlv, nops;
    size_t arr_off;          // byte offset of the level arrays in shared memory
    int arr_elems;           // elements of all level arrays (y follows them)
    size_t smem;             // dynamic shared memory bytes
    Terms<T> M;
    T omega;
    const T* lu;
    const int* piv;
    int nlu;
    Layout gL;               // entry level in global memory
    const T* gb;
    const T* gx_in;          // start iterate (entry_fz == 0)
    T* gx_out;               // result iterate
    int entry_fz, entry_a, out_a;
    int shape;               // SHAPE_* of M: named shapes get a compile-time term loop
};
template <class T> cudaError_t launch_tail(const TailArgs<T>& a, cudaStream_t s);
// cluster tail (kernels_tail.cu): middle levels on a thread-block cluster over their global
// buffers (ops with levels relative to the cluster entry level), TAIL_SOLO = the shared-memory
// tail in CTA 0 for entry (a_in, fz)
template <class T> struct ClusterArgs {
    const TailLevel<T>* lv;  // device array: the cluster levels and the first solo level (global buffers)
    const TailOp* ops;
    int nops;
    Terms<T> M;
    T omega;
    TailArgs<T> solo[2][2];
};
template <class T> cudaError_t launch_cluster_tail(const ClusterArgs<T>& a, int csize, size_t smem, cudaStream_t s);
template <class T> cudaError_t cluster_occupancy(int csize, size_t smem, int* nclusters);

}  // namespace spaimg
