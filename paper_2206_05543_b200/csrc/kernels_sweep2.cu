// Two smoothing steps in one 2D march (k_sweep2d_march Two = true): dispatch and instantiations.
#include "sweep2d_march.cuh"

namespace spaimg {

// ------------------------------------------------------------------------------------------
// two smoothing steps in one march (2D marching levels, named shapes): the second sweep runs
// three rows behind the first inside the same CTA (k_sweep2d_march TW), so x is read and x''
// written once per pair of sweeps: 24 B per unknown instead of 48.  no != nullptr: the norm of
// the INPUT residual is appended (part A); the K3 variant applies x + P e first.
// ------------------------------------------------------------------------------------------
// Used for the light stencils.  Measured on c2 (4095^2, fp64): jacobi2d V(2,2) 0.545 -> 0.483
// ms/cycle; the 9-point m9 pair is instruction-issue bound (58 % issue slots busy at 35 % of DRAM
// bandwidth, 135.8 us per pair against 2 x 66.6 us for two single-sweep marches), so BOX9 keeps
// one sweep per march and is not instantiated.
bool sweep2_supported(const Layout& L, int shape) {
    return L.dim == 2 && L.N > flat_threshold(2) && (shape == SHAPE_C1 || shape == SHAPE_STAR5);
}

template <class T, int S>
static cudaError_t sweep2_s(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA, T sM, T omega,
                            bool fz, const NormOut* no, cudaStream_t s) {
    const NormOut n0{};
    if (no)
        return fz ? launch_sweep2d_march<T, S, true, 1, true>(L, x, b, xo, M, sA, sM, omega, *no, s)
                  : launch_sweep2d_march<T, S, false, 1, true>(L, x, b, xo, M, sA, sM, omega, *no, s);
    return fz ? launch_sweep2d_march<T, S, true, 0, true>(L, x, b, xo, M, sA, sM, omega, n0, s)
              : launch_sweep2d_march<T, S, false, 0, true>(L, x, b, xo, M, sA, sM, omega, n0, s);
}

template <class T>
cudaError_t launch_sweep2(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, int shape, T sA, T sM,
                          T omega, bool from_zero, cudaStream_t s, const NormOut* no) {
    switch (shape) {
        case SHAPE_C1: return sweep2_s<T, SHAPE_C1>(L, x, b, xo, M, sA, sM, omega, from_zero, no, s);
        case SHAPE_STAR5: return sweep2_s<T, SHAPE_STAR5>(L, x, b, xo, M, sA, sM, omega, from_zero, no, s);
        default: return cudaErrorNotSupported;
    }
}

template <class T>
cudaError_t launch_sweep2_pc(const Layout& L, const Layout& Lc, const T* x, const T* e, const T* b, T* xo,
                             const Terms<T>& M, int shape, T sA, T sM, T omega, cudaStream_t s) {
    const NormOut none{};
    switch (shape) {
        case SHAPE_C1:
            return launch_sweep2d_march<T, SHAPE_C1, false, 3, true>(L, x, b, xo, M, sA, sM, omega, none, s, e, &Lc);
        case SHAPE_STAR5:
            return launch_sweep2d_march<T, SHAPE_STAR5, false, 3, true>(L, x, b, xo, M, sA, sM, omega, none, s, e,
                                                                       &Lc);
        default: return cudaErrorNotSupported;
    }
}

template cudaError_t launch_sweep2<double>(const Layout&, const double*, const double*, double*, const Terms<double>&,
                                           int, double, double, double, bool, cudaStream_t, const NormOut*);
template cudaError_t launch_sweep2<float>(const Layout&, const float*, const float*, float*, const Terms<float>&, int,
                                          float, float, float, bool, cudaStream_t, const NormOut*);
template cudaError_t launch_sweep2_pc<double>(const Layout&, const Layout&, const double*, const double*,
                                              const double*, double*, const Terms<double>&, int, double, double, double,
                                              cudaStream_t);
template cudaError_t launch_sweep2_pc<float>(const Layout&, const Layout&, const float*, const float*, const float*,
                                             float*, const Terms<float>&, int, float, float, float, cudaStream_t);

}  // namespace spaimg
