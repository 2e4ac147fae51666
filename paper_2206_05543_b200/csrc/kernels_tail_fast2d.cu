// K5+ fast path instantiations, 2D: entry level n = 63 (mesh count 64), coarse level
// n = 1 or 3 (coarsest_N = 2 or 4), the named smoother shapes.  See kernels_tail_fast.cuh.
#include "kernels_tail_fast.cuh"

namespace spaimg {

template <class T>
cudaError_t launch_tail_fast2d(const TailArgs<T>& a, cudaStream_t s) {
    if (a.fast_le != 6 || (a.fast_lc != 1 && a.fast_lc != 2)) return cudaErrorNotSupported;
    switch (a.shape) {
        case SHAPE_C1:
            return a.fast_lc == 1 ? launch_tail_fast_s<T, SHAPE_C1, 2, 6, 1>(a, s)
                                  : launch_tail_fast_s<T, SHAPE_C1, 2, 6, 2>(a, s);
        case SHAPE_STAR5:
            return a.fast_lc == 1 ? launch_tail_fast_s<T, SHAPE_STAR5, 2, 6, 1>(a, s)
                                  : launch_tail_fast_s<T, SHAPE_STAR5, 2, 6, 2>(a, s);
        case SHAPE_BOX9:
            return a.fast_lc == 1 ? launch_tail_fast_s<T, SHAPE_BOX9, 2, 6, 1>(a, s)
                                  : launch_tail_fast_s<T, SHAPE_BOX9, 2, 6, 2>(a, s);
        default: return cudaErrorNotSupported;
    }
}

template cudaError_t launch_tail_fast2d<double>(const TailArgs<double>&, cudaStream_t);
template cudaError_t launch_tail_fast2d<float>(const TailArgs<float>&, cudaStream_t);

}  // namespace spaimg
