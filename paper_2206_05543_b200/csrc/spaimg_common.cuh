// Shared device-side definitions for the spaimg B200 hot path.
//
// Arithmetic contract: every per-point expression reproduces the
// reference numpy expression tree with one IEEE rounding per operation and NO contraction,
// hence the explicit __d*_rn / __f*_rn intrinsics everywhere (the build also passes
// --fmad=false as a backstop).  Reference: pkg/src/spaimg/stencils.py:136-153 (apply),
// multigrid.py:86-101 (smooth), :104-119 (restrict), :122-144 (prolong), :176-184 (cycle).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace spaimg {

// ------------------------------------------------------------------------------------------
// checked build (SPAIMG_DEBUG_CHECKS -> libspaimg_cuda_debug.so, loaded with SPAIMG_DEBUG=1):
// the in-house stand-in for compute-sanitizer, which is closed on the GPU pool.
//   * SPAIMG_JITTER(): a random per-warp delay at every synchronisation point of the marching
//     kernels (mbarrier waits) and the coarse engines (op barriers), so a missing barrier or
//     wait shows up as a nondeterministic, non-bitwise result;
//   * level buffers and the engines' shared arrays start with NaN interiors and slack (zero
//     frames only), so any read before write or outside the stencil's reach poisons a result.
// ------------------------------------------------------------------------------------------
#ifdef SPAIMG_DEBUG_CHECKS
__device__ __forceinline__ void dbg_jitter() {
    const unsigned c = (unsigned)clock();
    const unsigned h = (c ^ ((threadIdx.x >> 5) * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu)) * 0xC2B2AE35u;
    if ((h >> 28) < 6) __nanosleep((h >> 8) & 1023u);
}
#define SPAIMG_JITTER() ::spaimg::dbg_jitter()
constexpr bool kDebugChecks = true;
#else
#define SPAIMG_JITTER() \
    do {                \
    } while (0)
constexpr bool kDebugChecks = false;
#endif

// ------------------------------------------------------------------------------------------
// rounding-exact scalar ops
// ------------------------------------------------------------------------------------------
template <class T> struct Op;
template <> struct Op<double> {
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
    static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
};
template <> struct Op<float> {
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
    static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
};

// ------------------------------------------------------------------------------------------
// padded level layout ("ghost frame"): every level of the hierarchy lives in a zero-framed,
// pitched array so that stencil loads never need bounds checks (the frame IS the reference's
// zero extension, stencils.py:139-146) and every row starts 128-byte aligned.
//   2D: rows [-2, n+2), columns [-LX, px-LX);      element (i0,i1)    at origin + i0*px + i1
//   3D: planes [-2, n+2), rows [-2, ry-2), cols ... element (i0,i1,i2) at origin + i0*pp + i1*px + i2
// Kernels only ever WRITE interior points, so the frame stays zero once cleared.
// ------------------------------------------------------------------------------------------
struct Layout {
    int dim;       // 2 or 3
    int N;         // mesh count; interior n = N-1 per axis
    int n;
    int esize;     // bytes per element (8 or 4)
    int ghost;     // zero frame rows/planes on each side (>= kGhost; >= the smoother's radius)
    long long px;  // row pitch (elements)
    long long pp;  // plane pitch (elements), 3D only
    long long origin;  // element offset of interior (0,0[,0])
    long long alloc;   // total elements
};

// tile extents the layout guarantees as addressable slack past the interior
constexpr int kTileX2D = 512;   // widest 2D strip (columns)
constexpr int kTileX3D = 128;   // widest 3D tile (columns)
constexpr int kTileY3D = 32;    // tallest 3D tile (rows)
constexpr int kGhost = 2;       // minimum ghost rows/planes (Layout::ghost) on the marching axes

// ------------------------------------------------------------------------------------------
// stencil term list (entries order of the reference dict, stencils.py:149-151)
// ------------------------------------------------------------------------------------------
constexpr int kMaxTerms = 27;
template <class T> struct Terms {
    int nt;
    int off[kMaxTerms][3];   // axis0, axis1, axis2 offsets, each in [-1, 1] for the fused kernels
    T c[kMaxTerms];          // float(c) rounded once to T
};

// shape classes with compile-time offsets (coefficients stay runtime); GENERIC reads offsets
// from the kernel parameters.
enum Shape : int {
    SHAPE_GENERIC = 0,
    SHAPE_C1 = 1,      // centre only (jacobi2d, jacobi3d)
    SHAPE_STAR5 = 2,   // 2D centre, (1,0),(-1,0),(0,1),(0,-1)       (m5tw, m5, laplacian order)
    SHAPE_BOX9 = 3,    // 2D STAR5 then (1,1),(1,-1),(-1,1),(-1,-1)  (vanka9, m9: upsilon order)
    SHAPE_STAR7 = 4,   // 3D centre, +-axis0, +-axis1, +-axis2       (m7, tee order)
};

template <int S> struct ShapeT;
template <> struct ShapeT<SHAPE_C1> {
    static constexpr int nt = 1;
    __host__ __device__ static constexpr int o(int, int) { return 0; }
};
template <> struct ShapeT<SHAPE_STAR5> {
    static constexpr int nt = 5;
    __host__ __device__ static constexpr int o(int k, int a) {
        // (0,0) (1,0) (-1,0) (0,1) (0,-1)
        return a == 0 ? (k == 1 ? 1 : k == 2 ? -1 : 0) : a == 1 ? (k == 3 ? 1 : k == 4 ? -1 : 0) : 0;
    }
};
template <> struct ShapeT<SHAPE_BOX9> {
    static constexpr int nt = 9;
    __host__ __device__ static constexpr int o(int k, int a) {
        // (0,0) (1,0) (-1,0) (0,1) (0,-1) (1,1) (1,-1) (-1,1) (-1,-1)
        return a == 0 ? (k == 1 ? 1 : k == 2 ? -1 : (k == 5 || k == 6) ? 1 : (k == 7 || k == 8) ? -1 : 0)
             : a == 1 ? (k == 3 ? 1 : k == 4 ? -1 : (k == 5 || k == 7) ? 1 : (k == 6 || k == 8) ? -1 : 0)
             : 0;
    }
};
template <> struct ShapeT<SHAPE_STAR7> {
    static constexpr int nt = 7;
    __host__ __device__ static constexpr int o(int k, int a) {
        // (0,0,0) (1,0,0) (-1,0,0) (0,1,0) (0,-1,0) (0,0,1) (0,0,-1)
        return k == 0 ? 0 : ((k - 1) / 2 == a ? ((k - 1) % 2 == 0 ? 1 : -1) : 0);
    }
};

// Device-side residual-history sink of the fused norm (see march.cuh norm_epilogue).
// Stop test of the reference solve loop (multigrid.py:211-217) evaluated on the device.
struct SolveCtl {
    double tol;
    int max_iters;
    int pad;
};

struct NormOut {
    double* partials;   // >= number of CTAs
    unsigned* counter;  // zero on entry, re-armed to zero by the last CTA
    double* norms;      // residual history
    int* slot;          // history cursor
    // optional (ctl != nullptr): the last CTA also runs the stop test on the new norm and sets
    // the solve loop's WHILE condition (state = {cycles done, converged})
    const SolveCtl* ctl;
    int* state;
    cudaGraphConditionalHandle cond;
};

// ------------------------------------------------------------------------------------------
// per-point expression trees
// ------------------------------------------------------------------------------------------

// A x at one interior point for the re-discretized Laplacian (stencils.py:209-223), scaled
// (stencils.py:152), then r = b - (A x) (multigrid.py:99).  Products by -1 are exact, so
// acc + (-1 (x) v) == acc - v bit for bit.
template <class T>
__device__ __forceinline__ T residual2d(T b, T xc, T xs, T xn, T xe, T xw, T sA) {
    using O = Op<T>;
    // (0,0):4  (1,0):-1  (-1,0):-1  (0,1):-1  (0,-1):-1
    T acc = O::add(T(0), O::mul(T(4), xc));
    acc = O::sub(acc, xs);   // (1,0):  next row along axis 0
    acc = O::sub(acc, xn);   // (-1,0): previous row
    acc = O::sub(acc, xe);   // (0,1)
    acc = O::sub(acc, xw);   // (0,-1)
    return O::sub(b, O::mul(acc, sA));
}

template <class T>
__device__ __forceinline__ T residual3d(T b, T xc, T xp0, T xm0, T xp1, T xm1, T xp2, T xm2, T sA) {
    using O = Op<T>;
    T acc = O::add(T(0), O::mul(T(6), xc));
    acc = O::sub(acc, xp0);
    acc = O::sub(acc, xm0);
    acc = O::sub(acc, xp1);
    acc = O::sub(acc, xm1);
    acc = O::sub(acc, xp2);
    acc = O::sub(acc, xm2);
    return O::sub(b, O::mul(acc, sA));
}

// x' = x + omega * ((sum_k c_k r_k) * sM)  (multigrid.py:100, stencils.py:149-152)
template <class T>
__device__ __forceinline__ T relax(T x, T accM, T sM, T omega) {
    using O = Op<T>;
    return O::add(x, O::mul(omega, O::mul(accM, sM)));
}

// full weighting of one line triple (multigrid.py:106): (0.25 a + 0.5 b) + 0.25 c
template <class T>
__device__ __forceinline__ T fw(T a, T b, T c) {
    using O = Op<T>;
    return O::add(O::add(O::mul(T(0.25), a), O::mul(T(0.5), b)), O::mul(T(0.25), c));
}

// prolongation value of fine line index i from coarse line values (multigrid.py:126-129):
// odd i -> a[i/2]; even interior 2j -> 0.5 (a[j-1] + a[j]); ends 0.5 a[0] and 0.5 a[m-1].
template <class T>
__device__ __forceinline__ T pl_even(T am1, T a0, bool first, bool last) {
    using O = Op<T>;
    // one multiply for all three cases (the same values bit for bit: only the operand differs)
    const T s = first ? a0 : (last ? am1 : O::add(am1, a0));
    return O::mul(T(0.5), s);
}

}  // namespace spaimg
