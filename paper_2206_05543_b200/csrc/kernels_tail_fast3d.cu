// K5+ fast path instantiations, 3D: entry level n = 15 (mesh count 16), coarse level
// n = 1 or 3 (coarsest_N = 2 or 4), the named smoother shapes.  See kernels_tail_fast.cuh.
#include "kernels_tail_fast.cuh"

namespace spaimg {

template <class T>
cudaError_t launch_tail_fast3d(const TailArgs<T>& a, cudaStream_t s) {
    if (a.fast_le != 4 || (a.fast_lc != 1 && a.fast_lc != 2)) return cudaErrorNotSupported;
    switch (a.shape) {
        case SHAPE_C1:
            return a.fast_lc == 1 ? launch_tail_fast_s<T, SHAPE_C1, 3, 4, 1>(a, s)
                                  : launch_tail_fast_s<T, SHAPE_C1, 3, 4, 2>(a, s);
        case SHAPE_STAR7:
            return a.fast_lc == 1 ? launch_tail_fast_s<T, SHAPE_STAR7, 3, 4, 1>(a, s)
                                  : launch_tail_fast_s<T, SHAPE_STAR7, 3, 4, 2>(a, s);
        default: return cudaErrorNotSupported;
    }
}

template cudaError_t launch_tail_fast3d<double>(const TailArgs<double>&, cudaStream_t);
template cudaError_t launch_tail_fast3d<float>(const TailArgs<float>&, cudaStream_t);

}  // namespace spaimg
