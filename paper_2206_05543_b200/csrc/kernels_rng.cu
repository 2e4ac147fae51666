// Device-side numpy Generator(PCG64).uniform(low, high, size) draws, bitwise:
// the reference solve() starts from default_rng(rng_seed).uniform(0, 1, shape) (reference
// multigrid.py:204-205).  Drawing it on the host costs a numpy pass plus a host->device copy of the
// whole vector (1 GB at 511^3); here the host only seeds (SeedSequence -> PCG64 state, numpy) and
// every thread jumps the 128-bit LCG ahead to its first element.
//   step:   s <- s * M + inc  (mod 2^128), M = numpy's PCG_DEFAULT_MULTIPLIER_128
//   output: rotr64(hi ^ lo, hi >> 58) of the stepped state  (XSL-RR)
//   double: (u64 >> 11) * 2^-53;  uniform = low + (high - low) * double
#include <cstdint>

#include "kernels.h"

namespace spaimg {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 pcg_mult() {
    return ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
}

// state after `delta` steps (pcg_advance_lcg_128)
__device__ __forceinline__ u128 pcg_advance(u128 state, unsigned long long delta, u128 inc) {
    u128 am = 1, ap = 0, cm = pcg_mult(), cp = inc;
    while (delta) {
        if (delta & 1) {
            am *= cm;
            ap = ap * cm + cp;
        }
        cp = (cm + 1) * cp;
        cm *= cm;
        delta >>= 1;
    }
    return am * state + ap;
}

__device__ __forceinline__ double pcg_next_double(u128& s, u128 inc) {
    s = s * pcg_mult() + inc;
    const unsigned long long hi = (unsigned long long)(s >> 64), lo = (unsigned long long)s;
    const unsigned long long x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    const unsigned long long u = (x >> r) | (x << ((64 - r) & 63));
    return __dmul_rn((double)(u >> 11), 1.0 / 9007199254740992.0);
}

template <class T>
__global__ void k_fill_uniform(T* out, long long count, unsigned long long s_hi, unsigned long long s_lo,
                               unsigned long long i_hi, unsigned long long i_lo, double low, double high, int per) {
    const long long first = (blockIdx.x * (long long)blockDim.x + threadIdx.x) * per;
    if (first >= count) return;
    const u128 inc = ((u128)i_hi << 64) | i_lo;
    u128 s = pcg_advance(((u128)s_hi << 64) | s_lo, (unsigned long long)first, inc);
    const double span = __dsub_rn(high, low);
    const long long last = first + per < count ? first + per : count;
    for (long long i = first; i < last; ++i) {
        const double d = __dadd_rn(low, __dmul_rn(span, pcg_next_double(s, inc)));
        out[i] = (T)d;  // fp32 grids: the float64 draw rounded once, as numpy's astype / torch's .to
    }
}

template <class T>
cudaError_t launch_fill_uniform(T* out, long long count, const unsigned long long st[4], double low, double high,
                                cudaStream_t s) {
    if (count <= 0) return cudaSuccess;
    const int per = 64;  // elements per thread: one jump-ahead, then sequential steps
    const long long threads = (count + per - 1) / per;
    const long long blocks = (threads + 255) / 256;
    k_fill_uniform<T><<<(unsigned)blocks, 256, 0, s>>>(out, count, st[0], st[1], st[2], st[3], low, high, per);
    return cudaGetLastError();
}

template cudaError_t launch_fill_uniform<double>(double*, long long, const unsigned long long[4], double, double,
                                                 cudaStream_t);
template cudaError_t launch_fill_uniform<float>(float*, long long, const unsigned long long[4], double, double,
                                                cudaStream_t);

}  // namespace spaimg
