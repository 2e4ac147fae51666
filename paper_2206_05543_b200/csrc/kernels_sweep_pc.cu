// K3 + K1: the prolongation + correction fused into the first post-sweep (multigrid.py:184-185):
// dispatch and instantiations of the K3 + K1 marches (2D row march Mode 3, 3D plane march Mode 4).
#include "sweep2d_march.cuh"

namespace spaimg {

template <class T, int S, bool FZ, int NM>
cudaError_t launch_sweep3d_march(const Layout& L, const T* x, const T* b, T* xo, const Terms<T>& M, T sA, T sM,
                                 T omega, const NormOut& no, cudaStream_t s, const Layout* Lc = nullptr,
                                 const T* ec = nullptr);

// K3 + K1 fused: xo = sweep(x + P e) for the first post-smoothing step (multigrid.py:184-185),
// on 2D marching levels: the marching kernel with the correction applied to every staged x row
// (NM == 3).  Measured (tools/tune.py): a net win on the 4096^2 level (-16 B/unknown of HBM
// traffic; c2 m9 V(1,1) 0.385 -> 0.374 ms/cycle, jacobi2d 0.369 -> 0.337) and neutral on 2048^2
// and below, where its extra per-step work is not hidden once the level's HBM time is short.
// (A flat-tile fusion for the small levels was measured neutral in 2D and a loss in 3D, and
// removed.)
// 3D (plane march, named shapes): the prolonged iterate never goes to HBM, 25 B/unknown instead
// of 17 + 24.  SPAIMG_PC3_N sets the smallest 3D mesh count that uses it (0 turns it off).
static int pc3_min_n() {
    const char* e = getenv("SPAIMG_PC3_N");  // read per solver plan (host side, not per launch in a graph)
    return e ? atoi(e) : 256;
}
// SPAIMG_PC2_N: the smallest 2D mesh count that uses the fused march (default 4096; the level
// must be a marching level)
static int pc2_min_n() {
    const char* e = getenv("SPAIMG_PC2_N");
    return e ? atoi(e) : 4096;
}
bool sweep_pc_supported(const Layout& L, int shape) {
    if (L.dim == 2) return pc2_min_n() > 0 && L.N >= pc2_min_n() && L.N > flat_threshold(2);
    return pc3_min_n() > 0 && L.N >= pc3_min_n() && L.N > flat_threshold(3) && (shape == SHAPE_C1 || shape == SHAPE_STAR7);
}

template <class T>
cudaError_t launch_sweep_pc(const Layout& L, const Layout& Lc, const T* x, const T* e, const T* b, T* xo,
                            const Terms<T>& M, int shape, T sA, T sM, T omega, cudaStream_t s) {
    const NormOut none{};
    if (L.dim == 3) {
        if (shape == SHAPE_C1)
            return launch_sweep3d_march<T, SHAPE_C1, false, 4>(L, x, b, xo, M, sA, sM, omega, none, s, &Lc, e);
        if (shape == SHAPE_STAR7)
            return launch_sweep3d_march<T, SHAPE_STAR7, false, 4>(L, x, b, xo, M, sA, sM, omega, none, s, &Lc, e);
        return cudaErrorNotSupported;
    }
    switch (shape) {
        case SHAPE_C1: return launch_sweep2d_march<T, SHAPE_C1, false, 3>(L, x, b, xo, M, sA, sM, omega, none, s, e, &Lc);
        case SHAPE_STAR5:
            return launch_sweep2d_march<T, SHAPE_STAR5, false, 3>(L, x, b, xo, M, sA, sM, omega, none, s, e, &Lc);
        case SHAPE_BOX9:
            return launch_sweep2d_march<T, SHAPE_BOX9, false, 3>(L, x, b, xo, M, sA, sM, omega, none, s, e, &Lc);
        default:
            return launch_sweep2d_march<T, SHAPE_GENERIC, false, 3>(L, x, b, xo, M, sA, sM, omega, none, s, e, &Lc);
    }
}

template cudaError_t launch_sweep_pc<double>(const Layout&, const Layout&, const double*, const double*,
                                             const double*, double*, const Terms<double>&, int, double, double, double,
                                             cudaStream_t);
template cudaError_t launch_sweep_pc<float>(const Layout&, const Layout&, const float*, const float*, const float*,
                                            float*, const Terms<float>&, int, float, float, float, cudaStream_t);

}  // namespace spaimg
