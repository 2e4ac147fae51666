// Basic (per-point) sm_100a kernels of the spaimg hot path and their launchers:
// layout conversion, the generic stencil product (K0), the unfused residual / relax /
// restriction building blocks, prolongation+correction (K3), the deterministic residual
// norm (K4) and the coarse direct solve (K5).
//
// Every arithmetic expression is the Appendix-A tree of the reference numpy code; see
// spaimg_common.cuh for the cited reference lines.
#include <cmath>

#include <algorithm>

#include "kernels.h"
#include "march.cuh"

namespace spaimg {

// ------------------------------------------------------------------------------------------
// layout
// ------------------------------------------------------------------------------------------
static long long roundup(long long a, long long b) { return (a + b - 1) / b * b; }

Layout make_layout(int dim, int N, int esize, int ghost) {
    Layout L{};
    L.dim = dim;
    L.N = N;
    L.n = N - 1;
    L.esize = esize;
    const long long g = ghost < kGhost ? kGhost : ghost;
    L.ghost = (int)g;
    const long long n = N - 1;
    const long long LX = roundup(g, 128 / esize);        // interior column 0 is 128-byte aligned
    const long long V = std::max<long long>(16 / esize, g);  // right frame: 16-byte halo granule, >= ghost
    if (dim == 2) {
        L.px = roundup(LX + roundup(n, kTileX2D) + V, 32);
        const long long rows = n + 2 * g;
        L.pp = 0;
        L.origin = g * L.px + LX;
        L.alloc = rows * L.px;
    } else {
        L.px = roundup(LX + roundup(n, kTileX3D) + V, 32);
        const long long ry = g + roundup(n, kTileY3D) + g;
        L.pp = ry * L.px;
        const long long planes = n + 2 * g;
        L.origin = g * L.pp + g * L.px + LX;
        L.alloc = planes * L.pp;
    }
    return L;
}

__device__ __forceinline__ long long pidx(const Layout& L, int i0, int i1, int i2) {
    return L.dim == 2 ? L.origin + (long long)i0 * L.px + i1
                      : L.origin + (long long)i0 * L.pp + (long long)i1 * L.px + i2;
}

static dim3 pgrid(const Layout& L, int bx) {
    return L.dim == 2 ? dim3((L.n + bx - 1) / bx, L.n, 1) : dim3((L.n + bx - 1) / bx, L.n, L.n);
}

// ------------------------------------------------------------------------------------------
// pad / unpad
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_pad(Layout L, const T* __restrict__ dense, T* __restrict__ padded) {
    const int i2d = blockIdx.x * blockDim.x + threadIdx.x;
    if (i2d >= L.n) return;
    const long long n = L.n;
    if (L.dim == 2) {
        const int i0 = blockIdx.y;
        padded[pidx(L, i0, i2d, 0)] = dense[i0 * n + i2d];
    } else {
        const int i0 = blockIdx.z, i1 = blockIdx.y;
        padded[pidx(L, i0, i1, i2d)] = dense[(i0 * n + i1) * n + i2d];
    }
}

template <class T>
__global__ void k_unpad(Layout L, const T* __restrict__ padded, T* __restrict__ dense) {
    const int i2d = blockIdx.x * blockDim.x + threadIdx.x;
    if (i2d >= L.n) return;
    const long long n = L.n;
    if (L.dim == 2) {
        const int i0 = blockIdx.y;
        dense[i0 * n + i2d] = padded[pidx(L, i0, i2d, 0)];
    } else {
        const int i0 = blockIdx.z, i1 = blockIdx.y;
        dense[(i0 * n + i1) * n + i2d] = padded[pidx(L, i0, i1, i2d)];
    }
}

template <class T> cudaError_t launch_pad(const Layout& L, const T* dense, T* padded, cudaStream_t s) {
    k_pad<T><<<pgrid(L, 256), 256, 0, s>>>(L, dense, padded);
    return cudaGetLastError();
}
template <class T> cudaError_t launch_unpad(const Layout& L, const T* padded, T* dense, cudaStream_t s) {
    k_unpad<T><<<pgrid(L, 256), 256, 0, s>>>(L, padded, dense);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K0: generic zero-extended stencil product on dense arrays (stencils.py:136-153)
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_apply_dense(int dim, int n, const T* __restrict__ x, T* __restrict__ out, Terms<T> S, T scale) {
    using O = Op<T>;
    const long long nn = n;
    const long long cnt = dim == 2 ? nn * nn : nn * nn * nn;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < cnt;
         idx += (long long)gridDim.x * blockDim.x) {
        int i0, i1, i2 = 0;
        if (dim == 2) {
            i0 = (int)(idx / nn);
            i1 = (int)(idx % nn);
        } else {
            i0 = (int)(idx / (nn * nn));
            i1 = (int)((idx / nn) % nn);
            i2 = (int)(idx % nn);
        }
        T acc = T(0);
        for (int k = 0; k < S.nt; ++k) {
            const int j0 = i0 + S.off[k][0], j1 = i1 + S.off[k][1], j2 = i2 + S.off[k][2];
            T v = T(0);
            if (j0 >= 0 && j0 < n && j1 >= 0 && j1 < n && (dim == 2 || (j2 >= 0 && j2 < n)))
                v = dim == 2 ? x[j0 * nn + j1] : x[(j0 * nn + j1) * nn + j2];
            acc = O::add(acc, O::mul(S.c[k], v));
        }
        out[idx] = O::mul(acc, scale);
    }
}

template <class T>
cudaError_t launch_apply_dense(int dim, int N, const T* x, T* out, const Terms<T>& terms, T scale, cudaStream_t s) {
    const long long n = N - 1;
    const long long cnt = dim == 2 ? n * n : n * n * n;
    long long blocks = (cnt + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    k_apply_dense<T><<<(unsigned)blocks, 256, 0, s>>>(dim, N - 1, x, out, terms, scale);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// unfused residual r = b - A x on padded levels (r's frame stays zero)
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_residual(Layout L, const T* __restrict__ x, const T* __restrict__ b, T* __restrict__ r, T sA) {
    const int i2d = blockIdx.x * blockDim.x + threadIdx.x;
    if (i2d >= L.n) return;
    if (L.dim == 2) {
        const long long p = pidx(L, blockIdx.y, i2d, 0);
        r[p] = residual2d<T>(b[p], x[p], x[p + L.px], x[p - L.px], x[p + 1], x[p - 1], sA);
    } else {
        const long long p = pidx(L, blockIdx.z, blockIdx.y, i2d);
        r[p] = residual3d<T>(b[p], x[p], x[p + L.pp], x[p - L.pp], x[p + L.px], x[p - L.px], x[p + 1], x[p - 1], sA);
    }
}

template <class T>
cudaError_t launch_residual(const Layout& L, const T* x, const T* b, T* r, T sA, cudaStream_t s) {
    k_residual<T><<<pgrid(L, 256), 256, 0, s>>>(L, x, b, r, sA);
    return cudaGetLastError();
}

// x' = x + omega M r  with the generic (runtime) term list; radius <= kGhost
template <class T>
__global__ void k_relax(Layout L, const T* __restrict__ x, const T* __restrict__ r, T* __restrict__ xo, Terms<T> M,
                        T sM, T omega) {
    using O = Op<T>;
    const int i2d = blockIdx.x * blockDim.x + threadIdx.x;
    if (i2d >= L.n) return;
    const long long p = L.dim == 2 ? pidx(L, blockIdx.y, i2d, 0) : pidx(L, blockIdx.z, blockIdx.y, i2d);
    T acc = T(0);
    for (int k = 0; k < M.nt; ++k) {
        const long long q = L.dim == 2 ? p + M.off[k][0] * L.px + M.off[k][1]
                                       : p + M.off[k][0] * L.pp + M.off[k][1] * L.px + M.off[k][2];
        acc = O::add(acc, O::mul(M.c[k], r[q]));
    }
    xo[p] = relax<T>(x ? x[p] : T(0), acc, sM, omega);
}

template <class T>
cudaError_t launch_relax(const Layout& L, const T* x, const T* r, T* xo, const Terms<T>& M, int, T sM, T omega,
                         cudaStream_t s) {
    k_relax<T><<<pgrid(L, 256), 256, 0, s>>>(L, x, r, xo, M, sM, omega);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// restriction of a padded fine residual (multigrid.py:104-119), separable, axis 0 first
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_restrict(Layout Lf, Layout Lc, const T* __restrict__ r, T* __restrict__ bc) {
    const int K = blockIdx.x * blockDim.x + threadIdx.x;
    if (K >= Lc.n) return;
    if (Lf.dim == 2) {
        const int I = blockIdx.y;
        // t[I, j] for j = 2K, 2K+1, 2K+2 (axis 0), then axis 1
        T t[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            const long long p = pidx(Lf, 2 * I + 1, 2 * K + q, 0);
            t[q] = fw<T>(r[p - Lf.px], r[p], r[p + Lf.px]);
        }
        bc[pidx(Lc, I, K, 0)] = fw<T>(t[0], t[1], t[2]);
    } else {
        const int I = blockIdx.z, J = blockIdx.y;
        T u[3];
#pragma unroll
        for (int qk = 0; qk < 3; ++qk) {
            T t[3];
#pragma unroll
            for (int qj = 0; qj < 3; ++qj) {
                const long long p = pidx(Lf, 2 * I + 1, 2 * J + qj, 2 * K + qk);
                t[qj] = fw<T>(r[p - Lf.pp], r[p], r[p + Lf.pp]);
            }
            u[qk] = fw<T>(t[0], t[1], t[2]);
        }
        bc[pidx(Lc, I, J, K)] = fw<T>(u[0], u[1], u[2]);
    }
}

template <class T>
cudaError_t launch_restrict(const Layout& Lf, const Layout& Lc, const T* r, T* bc, cudaStream_t s) {
    k_restrict<T><<<pgrid(Lc, 128), 128, 0, s>>>(Lf, Lc, r, bc);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K3: prolongation + correction, in place (multigrid.py:122-144, :184)
// ------------------------------------------------------------------------------------------
// One thread per coarse cell (I, J[, K]) produces the 2^d fine points (2I..2I+1, 2J..2J+1, ...)
// it owns (cells on the far side own only the fine points that exist).  The separable passes
// run axis 0 first exactly as the reference (axis-0 interpolants t, then axis 1 [, axis 2]);
// coarse values at J-1 / K-1 come from the neighbouring lane by shuffle, the zero frame of the
// coarse level supplies the boundary zeros, and the first/last flags keep the reference's
// 0.5*a[0] / 0.5*a[-1] end formulas bit for bit.  Fine rows move as 16-byte vectors.
template <class T>
__device__ __forceinline__ T pe(T am1, T a0, bool first, bool last) {
    return pl_even<T>(am1, a0, first, last);
}

// 2D: each thread owns C = 16 / (2 sizeof(T)) consecutive coarse cells (1 in fp64, 2 in fp32), so
// every fine row segment it writes is one 16-byte vector.
template <class T>
__global__ void __launch_bounds__(128) k_prolong_correct2d(Layout Lf, Layout Lc, const T* xi, T* xo,
                                                           const T* __restrict__ e, bool acc) {
    using O = Op<T>;
    constexpr int C = 16 / (2 * (int)sizeof(T));
    constexpr int V = 2 * C;  // fine columns per thread
    const int m = Lc.n;
    const int J0 = (blockIdx.x * blockDim.x + threadIdx.x) * C;
    const int I = blockIdx.y;
    const int lane = threadIdx.x & 31;
    // coarse rows I-1 (u) and I (d) at columns J0-1 .. J0+C-1 (frames are zero)
    const T* ec = e + Lc.origin + (long long)I * Lc.px + J0;
    T eu[C + 1], ed[C + 1];
#pragma unroll
    for (int k = 0; k < C; ++k) {
        eu[k + 1] = ec[k - Lc.px];
        ed[k + 1] = ec[k];
    }
    eu[0] = __shfl_up_sync(0xffffffffu, eu[C], 1);
    ed[0] = __shfl_up_sync(0xffffffffu, ed[C], 1);
    if (lane == 0) {
        eu[0] = ec[-Lc.px - 1];
        ed[0] = ec[-1];
    }
    if (J0 > m) return;
    const bool fI = I == 0, lI = I == m;
    const int nf = Lf.n;
    const long long off0 = Lf.origin + (long long)(2 * I) * Lf.px + 2 * J0;
    const bool full = 2 * J0 + V <= nf;  // every owned fine column is interior
    // all loads of the (possibly aliased, in-place) fine iterate first, then the stores
    T xv[2][V] = {};
    if (acc) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if (2 * I + h >= nf) break;
            const T* src = xi + off0 + (long long)h * Lf.px;
            if (full) {
                V16<T>::ld(src, xv[h]);
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (2 * J0 + v < nf) xv[h][v] = src[v];
            }
        }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        if (2 * I + h >= nf) break;
        // axis 0 at fine row 2I+h for coarse columns J0-1 .. J0+C-1, then axis 1
        T a[C + 1];
#pragma unroll
        for (int k = 0; k <= C; ++k) a[k] = h ? ed[k] : pe<T>(eu[k], ed[k], fI, lI);
        T o[V];
#pragma unroll
        for (int k = 0; k < C; ++k) {
            const int J = J0 + k;
            o[2 * k] = pe<T>(a[k], a[k + 1], J == 0, J == m);  // column 2J
            o[2 * k + 1] = a[k + 1];                          // column 2J+1
        }
        if (acc) {
#pragma unroll
            for (int v = 0; v < V; ++v) o[v] = O::add(xv[h][v], o[v]);
        }
        T* dst = xo + off0 + (long long)h * Lf.px;
        if (full) {
            V16<T>::st(dst, o);
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if (2 * J0 + v < nf) dst[v] = o[v];
        }
    }
}

// 3D: each thread owns C = 16 / (2 sizeof(T)) consecutive coarse cells along axis 2.
template <class T>
__global__ void __launch_bounds__(128) k_prolong_correct3d(Layout Lf, Layout Lc, const T* xi, T* xo,
                                                           const T* __restrict__ e, bool acc) {
    using O = Op<T>;
    constexpr int C = 16 / (2 * (int)sizeof(T));
    constexpr int V = 2 * C;
    const int m = Lc.n;
    const int K0 = (blockIdx.x * blockDim.x + threadIdx.x) * C;
    const int J = blockIdx.y, I = blockIdx.z;
    const int lane = threadIdx.x & 31;
    // c[di][dj][k]: coarse value at (I-1+di, J-1+dj, K0-1+k), k = 0..C (frames are zero)
    T c[2][2][C + 1];
    const T* ec = e + Lc.origin + (long long)I * Lc.pp + (long long)J * Lc.px + K0;
#pragma unroll
    for (int di = 0; di < 2; ++di)
#pragma unroll
        for (int dj = 0; dj < 2; ++dj) {
            const T* q = ec + (long long)(di - 1) * Lc.pp + (long long)(dj - 1) * Lc.px;
#pragma unroll
            for (int k = 0; k < C; ++k) c[di][dj][k + 1] = q[k];
            c[di][dj][0] = __shfl_up_sync(0xffffffffu, c[di][dj][C], 1);
            if (lane == 0) c[di][dj][0] = q[-1];
        }
    if (K0 > m) return;
    const bool fI = I == 0, lI = I == m, fJ = J == 0, lJ = J == m;
    const int nf = Lf.n;
    const bool full = 2 * K0 + V <= nf;
    // all loads of the (possibly aliased, in-place) fine iterate first, then the stores
    T xv[2][2][V] = {};
    if (acc) {
#pragma unroll
        for (int hi = 0; hi < 2; ++hi)
#pragma unroll
            for (int hj = 0; hj < 2; ++hj) {
                if (2 * I + hi >= nf || 2 * J + hj >= nf) continue;
                const T* src = xi + Lf.origin + (long long)(2 * I + hi) * Lf.pp + (long long)(2 * J + hj) * Lf.px + 2 * K0;
                if (full) {
                    V16<T>::ld(src, xv[hi][hj]);
                } else {
#pragma unroll
                    for (int v = 0; v < V; ++v)
                        if (2 * K0 + v < nf) xv[hi][hj][v] = src[v];
                }
            }
    }
#pragma unroll
    for (int hi = 0; hi < 2; ++hi) {
        if (2 * I + hi >= nf) break;
        // axis 0 at fine plane 2I+hi, coarse (J-1+dj, K0-1+k)
        T t[2][C + 1];
#pragma unroll
        for (int dj = 0; dj < 2; ++dj)
#pragma unroll
            for (int k = 0; k <= C; ++k) t[dj][k] = hi ? c[1][dj][k] : pe<T>(c[0][dj][k], c[1][dj][k], fI, lI);
#pragma unroll
        for (int hj = 0; hj < 2; ++hj) {
            if (2 * J + hj >= nf) break;
            // axis 1 at fine row 2J+hj, then axis 2
            T u[C + 1];
#pragma unroll
            for (int k = 0; k <= C; ++k) u[k] = hj ? t[1][k] : pe<T>(t[0][k], t[1][k], fJ, lJ);
            T o[V];
#pragma unroll
            for (int k = 0; k < C; ++k) {
                const int K = K0 + k;
                o[2 * k] = pe<T>(u[k], u[k + 1], K == 0, K == m);  // column 2K
                o[2 * k + 1] = u[k + 1];                          // column 2K+1
            }
            if (acc) {
#pragma unroll
                for (int v = 0; v < V; ++v) o[v] = O::add(xv[hi][hj][v], o[v]);
            }
            T* dst = xo + Lf.origin + (long long)(2 * I + hi) * Lf.pp + (long long)(2 * J + hj) * Lf.px + 2 * K0;
            if (full) {
                V16<T>::st(dst, o);
            } else {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (2 * K0 + v < nf) dst[v] = o[v];
            }
        }
    }
}

template <class T>
cudaError_t launch_prolong_correct(const Layout& Lf, const Layout& Lc, const T* xi, T* xo, const T* e, cudaStream_t s,
                                   bool acc) {
    const int m = Lc.n;
    if (Lf.dim == 2) {
        constexpr int C = 16 / (2 * (int)sizeof(T));
        dim3 g(((m + 1 + C - 1) / C + 127) / 128, m + 1);
        return launch_k(k_prolong_correct2d<T>, g, dim3(128), 0, s, Lf, Lc, xi, xo, e, acc);
    } else {
        constexpr int C = 16 / (2 * (int)sizeof(T));
        dim3 g(((m + 1 + C - 1) / C + 127) / 128, m + 1, m + 1);
        return launch_k(k_prolong_correct3d<T>, g, dim3(128), 0, s, Lf, Lc, xi, xo, e, acc);
    }
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K4: ||b - A x||_2, deterministic: fixed per-thread strides, fixed shuffle tree, fixed
// partial order in the last block (no floating-point atomics).
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <class T>
__global__ void __launch_bounds__(256) k_residual_norm(Layout L, const T* __restrict__ x, const T* __restrict__ b,
                                                       T sA, double* __restrict__ partials,
                                                       unsigned* __restrict__ counter, double* __restrict__ norms,
                                                       int slot, int* __restrict__ slot_dev) {
    __shared__ double red[8];
    __shared__ bool last;
    const long long n = L.n;
    const long long rows = L.dim == 2 ? n : n * n;
    double s = 0.0;
    // rows are distributed round-robin over blocks; threads stride within a row
    for (long long q = blockIdx.x; q < rows; q += gridDim.x) {
        const int i0 = L.dim == 2 ? (int)q : (int)(q / n);
        const int i1 = L.dim == 2 ? 0 : (int)(q % n);
        for (int k = threadIdx.x; k < L.n; k += blockDim.x) {
            T rv;
            if (L.dim == 2) {
                const long long p = pidx(L, i0, k, 0);
                rv = residual2d<T>(b[p], x[p], x[p + L.px], x[p - L.px], x[p + 1], x[p - 1], sA);
            } else {
                const long long p = pidx(L, i0, i1, k);
                rv = residual3d<T>(b[p], x[p], x[p + L.pp], x[p - L.pp], x[p + L.px], x[p - L.px], x[p + 1],
                                   x[p - 1], sA);
            }
            const double d = (double)rv;
            s = __dadd_rn(s, __dmul_rn(d, d));
        }
    }
    s = warp_sum(s);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (l == 0) red[w] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < (int)(blockDim.x >> 5); ++i) t += red[i];
        partials[blockIdx.x] = t;
        __threadfence();
        const unsigned done = atomicAdd(counter, 1u);
        last = (done == gridDim.x - 1);
    }
    __syncthreads();
    if (last && w == 0) {
        __threadfence();
        double t = 0.0;
        for (int i = l; i < (int)gridDim.x; i += 32) t += ((volatile double*)partials)[i];
        t = warp_sum(t);
        if (l == 0) {
            // slot_dev (if given) makes the kernel replayable in a graph: it appends to the
            // device-side residual history and advances the cursor.
            const int sl = slot_dev ? *slot_dev : slot;
            norms[sl] = sqrt(t);
            if (slot_dev) *slot_dev = sl + 1;
            *counter = 0u;  // re-arm for the next launch / graph replay
        }
    }
}

template <class T>
cudaError_t launch_residual_norm(const Layout& L, const T* x, const T* b, T sA, double* partials, unsigned* counter,
                                 double* norms, int slot, int* slot_dev, cudaStream_t s) {
    const long long rows = L.dim == 2 ? (long long)L.n : (long long)L.n * L.n;
    int blocks = (int)(rows < kNormBlocks ? rows : kNormBlocks);
    k_residual_norm<T><<<blocks, 256, 0, s>>>(L, x, b, sA, partials, counter, norms, slot, slot_dev);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// K5: coarse direct solve, getrs order (Appendix A.5 / A.6): row interchanges, column-oriented
// unit-lower forward substitution with FMA, column-oriented upper back substitution with a true
// division.  One CTA; each unknown is updated in the same j order as the sequential loop.
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_coarse_solve(Layout L, const T* __restrict__ b, T* __restrict__ x, const T* __restrict__ lu,
                               const int* __restrict__ piv, int nlu) {
    using O = Op<T>;
    extern __shared__ unsigned char smem_raw[];
    T* y = reinterpret_cast<T*>(smem_raw);
    const int n = L.n;
    for (int q = threadIdx.x; q < nlu; q += blockDim.x) {
        const int i0 = L.dim == 2 ? q / n : q / (n * n);
        const int i1 = L.dim == 2 ? q % n : (q / n) % n;
        const int i2 = L.dim == 2 ? 0 : q % n;
        y[q] = b[pidx(L, i0, i1, i2)];
    }
    __syncthreads();
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
    __syncthreads();
    for (int j = 0; j < nlu; ++j) {
        const T yj = y[j];
        for (int i = j + 1 + threadIdx.x; i < nlu; i += blockDim.x) y[i] = O::fma(-lu[(long long)i * nlu + j], yj, y[i]);
        __syncthreads();
    }
    for (int j = nlu - 1; j >= 0; --j) {
        if (threadIdx.x == 0) y[j] = O::div(y[j], lu[(long long)j * nlu + j]);
        __syncthreads();
        const T yj = y[j];
        for (int i = threadIdx.x; i < j; i += blockDim.x) y[i] = O::fma(-lu[(long long)i * nlu + j], yj, y[i]);
        __syncthreads();
    }
    for (int q = threadIdx.x; q < nlu; q += blockDim.x) {
        const int i0 = L.dim == 2 ? q / n : q / (n * n);
        const int i1 = L.dim == 2 ? q % n : (q / n) % n;
        const int i2 = L.dim == 2 ? 0 : q % n;
        x[pidx(L, i0, i1, i2)] = y[q];
    }
}

template <class T>
cudaError_t launch_coarse_solve(const Layout& L, const T* b, T* x, const T* lu, const int* piv, int nlu,
                                cudaStream_t s) {
    const size_t smem = (size_t)nlu * sizeof(T);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(k_coarse_solve<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    return launch_k(k_coarse_solve<T>, dim3(1), dim3(256), smem, s, L, b, x, lu, piv, nlu);
}

// ------------------------------------------------------------------------------------------
// checked build: a level buffer with NaN on its interior and on the slack beyond the two-cell
// zero frame (the frame itself zero), so every read the algorithm does not define poisons
// ------------------------------------------------------------------------------------------
template <class T>
__global__ void k_poison_level(Layout L, T* p) {
    const long long lx = L.origin % L.px;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < L.alloc;
         e += (long long)gridDim.x * blockDim.x) {
        long long i0, i1, i2 = 0;
        if (L.dim == 2) {
            i0 = e / L.px - L.ghost;
            i1 = e % L.px - lx;
        } else {
            const long long rem = e % L.pp;
            i0 = e / L.pp - L.ghost;
            i1 = rem / L.px - L.ghost;
            i2 = rem % L.px - lx;
        }
        auto in = [&](long long i, long long lo, long long hi) { return i >= lo && i < hi; };
        const long long n = L.n;
        const bool interior = in(i0, 0, n) && in(i1, 0, n) && (L.dim == 2 || in(i2, 0, n));
        const long long g = L.ghost;
        const bool frame = in(i0, -g, n + g) && in(i1, -g, n + g) && (L.dim == 2 || in(i2, -g, n + g));
        p[e] = (interior || !frame) ? T(__int_as_float(0x7fc00000)) : T(0);
    }
}

template <class T>
cudaError_t launch_poison_level(const Layout& L, T* p, cudaStream_t s) {
    k_poison_level<T><<<592, 256, 0, s>>>(L, p);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// explicit instantiations
// ------------------------------------------------------------------------------------------
#define SPAIMG_INST(T)                                                                                          \
    template cudaError_t launch_poison_level<T>(const Layout&, T*, cudaStream_t);                               \
    template cudaError_t launch_pad<T>(const Layout&, const T*, T*, cudaStream_t);                              \
    template cudaError_t launch_unpad<T>(const Layout&, const T*, T*, cudaStream_t);                            \
    template cudaError_t launch_apply_dense<T>(int, int, const T*, T*, const Terms<T>&, T, cudaStream_t);       \
    template cudaError_t launch_residual<T>(const Layout&, const T*, const T*, T*, T, cudaStream_t);            \
    template cudaError_t launch_relax<T>(const Layout&, const T*, const T*, T*, const Terms<T>&, int, T, T,     \
                                         cudaStream_t);                                                         \
    template cudaError_t launch_restrict<T>(const Layout&, const Layout&, const T*, T*, cudaStream_t);          \
    template cudaError_t launch_prolong_correct<T>(const Layout&, const Layout&, const T*, T*, const T*, cudaStream_t, bool); \
    template cudaError_t launch_residual_norm<T>(const Layout&, const T*, const T*, T, double*, unsigned*,      \
                                                 double*, int, int*, cudaStream_t);                             \
    template cudaError_t launch_coarse_solve<T>(const Layout&, const T*, T*, const T*, const int*, int,         \
                                                cudaStream_t);
SPAIMG_INST(double)
SPAIMG_INST(float)

}  // namespace spaimg
