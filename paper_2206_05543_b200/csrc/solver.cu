// C-ABI entry points (include/spaimg_cuda.h) and the native multigrid runtime: the padded
// level hierarchy, the V/W-cycle schedule (reference multigrid.py:157-185) captured into a
// CUDA graph, and the solve loop (multigrid.py:203-219).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "kernels.h"
#include "march.cuh"
#include "spaimg_cuda.h"

using namespace spaimg;

// ------------------------------------------------------------------------------------------
// errors
// ------------------------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CK(expr)                                                                                          \
    do {                                                                                                  \
        cudaError_t e_ = (expr);                                                                          \
        if (e_ != cudaSuccess) return fail((int)e_, std::string(#expr) + ": " + cudaGetErrorString(e_)); \
    } while (0)

extern "C" const char* spaimg_last_error(void) { return g_err.c_str(); }
extern "C" int spaimg_abi_version(void) { return SPAIMG_ABI_VERSION; }
extern "C" int spaimg_set_device(int device) {
    CK(cudaSetDevice(device));
    return 0;
}

// ------------------------------------------------------------------------------------------
// helpers
// ------------------------------------------------------------------------------------------
static bool is_device_ptr(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

static long long count_of(int dim, int N) {
    const long long n = N - 1;
    return dim == 2 ? n * n : n * n * n;
}

static int stencil_radius(const spaimg_stencil& S) {
    int w = 0;
    for (int k = 0; k < S.nterms; ++k)
        for (int a = 0; a < S.dim; ++a) w = std::max(w, std::abs(S.offsets[k][a]));
    return w;
}

static bool same_offsets(const spaimg_stencil& S, int shape) {
    auto o = [&](int k, int a) -> int {
        switch (shape) {
            case SHAPE_C1: return ShapeT<SHAPE_C1>::o(k, a);
            case SHAPE_STAR5: return ShapeT<SHAPE_STAR5>::o(k, a);
            case SHAPE_BOX9: return ShapeT<SHAPE_BOX9>::o(k, a);
            case SHAPE_STAR7: return ShapeT<SHAPE_STAR7>::o(k, a);
        }
        return 99;
    };
    int nt = shape == SHAPE_C1 ? 1 : shape == SHAPE_STAR5 ? 5 : shape == SHAPE_BOX9 ? 9 : 7;
    if (S.nterms != nt) return false;
    for (int k = 0; k < nt; ++k)
        for (int a = 0; a < S.dim; ++a)
            if (S.offsets[k][a] != o(k, a)) return false;
    return true;
}

static int detect_shape(const spaimg_stencil& S) {
    if (same_offsets(S, SHAPE_C1)) return SHAPE_C1;
    if (S.dim == 2 && same_offsets(S, SHAPE_STAR5)) return SHAPE_STAR5;
    if (S.dim == 2 && same_offsets(S, SHAPE_BOX9)) return SHAPE_BOX9;
    if (S.dim == 3 && same_offsets(S, SHAPE_STAR7)) return SHAPE_STAR7;
    return SHAPE_GENERIC;
}

template <class T>
static Terms<T> to_terms(const spaimg_stencil& S) {
    Terms<T> t{};
    t.nt = S.nterms;
    for (int k = 0; k < S.nterms; ++k) {
        for (int a = 0; a < 3; ++a) t.off[k][a] = a < S.dim ? S.offsets[k][a] : 0;
        t.c[k] = (T)S.coef[k];
    }
    return t;
}

// Python evaluates the mesh scale as (1.0 / N) ** e, i.e. C pow() (stencils.py:152)
static double hscale(int N, int e) { return std::pow(1.0 / (double)N, (double)e); }

static int check_stencil(const spaimg_stencil* S, int dim) {
    if (!S) return fail(SPAIMG_EINVAL, "stencil is NULL");
    if (S->dim != dim) return fail(SPAIMG_EINVAL, "stencil dim does not match grid dim");
    if (S->nterms < 1 || S->nterms > SPAIMG_MAX_TERMS) return fail(SPAIMG_EINVAL, "stencil needs 1..27 entries");
    return 0;
}

static int check_dims(int dtype, int dim, int N) {
    if (dtype != SPAIMG_F64 && dtype != SPAIMG_F32) return fail(SPAIMG_EINVAL, "dtype must be SPAIMG_F64 or SPAIMG_F32");
    if (dim != 2 && dim != 3) return fail(SPAIMG_EINVAL, "dim must be 2 or 3");
    if (N < 2) return fail(SPAIMG_EINVAL, "need N >= 2");
    return 0;
}

// A padded level with its buffers; owns cudaMalloc'd (or stream-ordered) memory.
template <class T> struct Level {
    Layout L{};
    T* x[2] = {nullptr, nullptr};
    T* b = nullptr;
    T* r = nullptr;  // scratch for unfused paths
    T sA{}, sM{};
};

// Stream-ordered scratch allocations for one-shot C-ABI calls.
struct Scratch {
    cudaStream_t s;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t st) : s(st) {}
    template <class T> cudaError_t get(T** p, size_t count) {
        void* q = nullptr;
        cudaError_t e = cudaMallocAsync(&q, count * sizeof(T), s);
        if (e != cudaSuccess) return e;
        ptrs.push_back(q);
        *p = static_cast<T*>(q);
        return cudaMemsetAsync(q, 0, count * sizeof(T), s);
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, s);
    }
};

// copy a dense input (host or device) into a padded level buffer
template <class T>
static int load_dense(Scratch& sc, const Layout& L, const void* src, T* padded, cudaStream_t s,
                      T* stage_buf = nullptr) {
    const long long cnt = count_of(L.dim, L.N);
    const T* dsrc = static_cast<const T*>(src);
    if (!is_device_ptr(src)) {
        T* stage = stage_buf;
        if (!stage) CK(sc.get(&stage, (size_t)cnt));
        CK(cudaMemcpyAsync(stage, src, (size_t)cnt * sizeof(T), cudaMemcpyHostToDevice, s));
        dsrc = stage;
    }
    CK(launch_pad<T>(L, dsrc, padded, s));
    return 0;
}

// copy a padded level buffer out to a dense destination (host or device)
template <class T>
static int store_dense(Scratch& sc, const Layout& L, const T* padded, void* dst, cudaStream_t s,
                       T* stage_buf = nullptr) {
    const long long cnt = count_of(L.dim, L.N);
    if (is_device_ptr(dst)) {
        CK(launch_unpad<T>(L, padded, static_cast<T*>(dst), s));
        return 0;
    }
    T* stage = stage_buf;
    if (!stage) CK(sc.get(&stage, (size_t)cnt));
    CK(launch_unpad<T>(L, padded, stage, s));
    CK(cudaMemcpyAsync(dst, stage, (size_t)cnt * sizeof(T), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return 0;
}

template <class T>
static int alloc_level(Scratch& sc, Level<T>& lv, int dim, int N, bool two_x, bool with_b, bool with_r,
                       int ghost = kGhost) {
    lv.L = make_layout(dim, N, sizeof(T), ghost);
    lv.sA = (T)hscale(N, -2);
    CK(sc.get(&lv.x[0], (size_t)lv.L.alloc));
    if (two_x) CK(sc.get(&lv.x[1], (size_t)lv.L.alloc));
    if (with_b) CK(sc.get(&lv.b, (size_t)lv.L.alloc));
    if (with_r) CK(sc.get(&lv.r, (size_t)lv.L.alloc));
    return 0;
}

// one smoothing step on a level: x[a] -> x[1-a]
template <class T>
static int do_sweep(Level<T>& lv, int a, bool fz, const Terms<T>& M, int shape, bool fused, T omega, cudaStream_t s,
                    int* launches) {
    if (fused) {
        CK(launch_sweep<T>(lv.L, lv.x[a], lv.b, lv.x[1 - a], M, shape, lv.sA, lv.sM, omega, fz, s));
        if (launches) *launches += 1;
        return 0;
    }
    if (fz) {
        CK(cudaMemsetAsync(lv.x[a], 0, (size_t)lv.L.alloc * sizeof(T), s));
        if (launches) *launches += 1;
    }
    CK(launch_residual<T>(lv.L, lv.x[a], lv.b, lv.r, lv.sA, s));
    CK(launch_relax<T>(lv.L, lv.x[a], lv.r, lv.x[1 - a], M, shape, lv.sM, omega, s));
    if (launches) *launches += 2;
    return 0;
}

// ------------------------------------------------------------------------------------------
// one-shot operator entry points
// ------------------------------------------------------------------------------------------
template <class T>
static int apply_t(int N, const spaimg_stencil* S, const void* x, void* out, cudaStream_t s) {
    Scratch sc(s);
    const int dim = S->dim;
    const long long cnt = count_of(dim, N);
    const T* dx = static_cast<const T*>(x);
    T* dout = static_cast<T*>(out);
    const bool host_out = !is_device_ptr(out);
    if (!is_device_ptr(x)) {
        T* st = nullptr;
        CK(sc.get(&st, (size_t)cnt));
        CK(cudaMemcpyAsync(st, x, (size_t)cnt * sizeof(T), cudaMemcpyHostToDevice, s));
        dx = st;
    }
    if (host_out) CK(sc.get(&dout, (size_t)cnt));
    CK(launch_apply_dense<T>(dim, N, dx, dout, to_terms<T>(*S), (T)hscale(N, S->h_exponent), s));
    if (host_out) {
        CK(cudaMemcpyAsync(out, dout, (size_t)cnt * sizeof(T), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    return 0;
}

extern "C" int spaimg_apply(int dtype, int N, const spaimg_stencil* S, const void* x, void* out, void* stream) {
    if (!S) return fail(SPAIMG_EINVAL, "stencil is NULL");
    if (int rc = check_dims(dtype, S->dim, N)) return rc;
    if (int rc = check_stencil(S, S->dim)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SPAIMG_F64 ? apply_t<double>(N, S, x, out, s) : apply_t<float>(N, S, x, out, s);
}

template <class T>
static int smooth_t(int dim, int N, const void* u, const void* b, const spaimg_stencil* Ms, double omega, int steps,
                    void* out, cudaStream_t s) {
    Scratch sc(s);
    Level<T> lv;
    const int rad = stencil_radius(*Ms);
    const int shape = detect_shape(*Ms);
    const bool fused = rad <= 1 && sweep_fused_supported(dim, shape);
    // the zero frame is as wide as the smoother's reach (stencils.py:139-146)
    if (int rc = alloc_level<T>(sc, lv, dim, N, true, true, !fused, std::max(kGhost, rad))) return rc;
    lv.sM = (T)hscale(N, Ms->h_exponent);
    if (int rc = load_dense<T>(sc, lv.L, u, lv.x[0], s)) return rc;
    if (steps > 0)
        if (int rc = load_dense<T>(sc, lv.L, b, lv.b, s)) return rc;
    const Terms<T> M = to_terms<T>(*Ms);
    int a = 0;
    for (int k = 0; k < steps;) {
        // pairs of steps in one march on the 2D marching sizes
        const bool pair = fused && steps - k >= 2 && sweep2_supported(lv.L, shape);
        if (pair) {
            CK(launch_sweep2<T>(lv.L, lv.x[a], lv.b, lv.x[1 - a], M, shape, lv.sA, lv.sM, (T)omega, false, s));
        } else if (int rc = do_sweep<T>(lv, a, false, M, shape, fused, (T)omega, s, nullptr)) {
            return rc;
        }
        k += pair ? 2 : 1;
        a = 1 - a;
    }
    return store_dense<T>(sc, lv.L, lv.x[a], out, s);
}

extern "C" int spaimg_smooth(int dtype, int dim, int N, const void* u, const void* b, const spaimg_stencil* M,
                             double omega, int steps, void* out, void* stream) {
    if (int rc = check_dims(dtype, dim, N)) return rc;
    if (int rc = check_stencil(M, dim)) return rc;
    if (steps < 0) return fail(SPAIMG_EINVAL, "steps must be non-negative");
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SPAIMG_F64 ? smooth_t<double>(dim, N, u, b, M, omega, steps, out, s)
                               : smooth_t<float>(dim, N, u, b, M, omega, steps, out, s);
}

static int check_halving(int N) {
    if (N % 2) return fail(SPAIMG_EINVAL, "cannot halve an odd mesh count N=" + std::to_string(N));
    if (N / 2 < 2) return fail(SPAIMG_EINVAL, "coarse mesh would have no interior points");
    return 0;
}

template <class T>
static int restrict_t(int dim, int N, const void* fine, void* coarse, cudaStream_t s) {
    Scratch sc(s);
    Level<T> f, c;
    if (int rc = alloc_level<T>(sc, f, dim, N, false, false, false)) return rc;
    if (int rc = alloc_level<T>(sc, c, dim, N / 2, false, false, false)) return rc;
    if (int rc = load_dense<T>(sc, f.L, fine, f.x[0], s)) return rc;
    CK(launch_restrict<T>(f.L, c.L, f.x[0], c.x[0], s));
    return store_dense<T>(sc, c.L, c.x[0], coarse, s);
}

extern "C" int spaimg_restrict(int dtype, int dim, int N, const void* fine, void* coarse, void* stream) {
    if (int rc = check_dims(dtype, dim, N)) return rc;
    if (int rc = check_halving(N)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SPAIMG_F64 ? restrict_t<double>(dim, N, fine, coarse, s) : restrict_t<float>(dim, N, fine, coarse, s);
}

template <class T>
static int prolong_t(int dim, int Nc, const void* coarse, const void* base, void* fine, cudaStream_t s) {
    Scratch sc(s);
    Level<T> f, c;
    if (int rc = alloc_level<T>(sc, f, dim, 2 * Nc, false, false, false)) return rc;
    if (int rc = alloc_level<T>(sc, c, dim, Nc, false, false, false)) return rc;
    if (int rc = load_dense<T>(sc, c.L, coarse, c.x[0], s)) return rc;
    if (base)
        if (int rc = load_dense<T>(sc, f.L, base, f.x[0], s)) return rc;
    // prolong(e) alone stores the interpolant (multigrid.py:125-129); with a base grid it is
    // the correction u + prolong(e) of multigrid.py:184.
    CK(launch_prolong_correct<T>(f.L, c.L, f.x[0], f.x[0], c.x[0], s, base != nullptr));
    return store_dense<T>(sc, f.L, f.x[0], fine, s);
}

extern "C" int spaimg_prolong(int dtype, int dim, int coarse_N, const void* coarse, void* fine, void* stream) {
    if (int rc = check_dims(dtype, dim, coarse_N)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SPAIMG_F64 ? prolong_t<double>(dim, coarse_N, coarse, nullptr, fine, s)
                               : prolong_t<float>(dim, coarse_N, coarse, nullptr, fine, s);
}

extern "C" int spaimg_prolong_correct(int dtype, int dim, int N, const void* u, const void* e, void* out, void* stream) {
    if (int rc = check_dims(dtype, dim, N)) return rc;
    if (int rc = check_halving(N)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SPAIMG_F64 ? prolong_t<double>(dim, N / 2, e, u, out, s)
                               : prolong_t<float>(dim, N / 2, e, u, out, s);
}

template <class T>
static int residual_restrict_t(int dim, int N, const void* u, const void* b, void* coarse, cudaStream_t s) {
    Scratch sc(s);
    Level<T> f, c;
    if (int rc = alloc_level<T>(sc, f, dim, N, false, true, false)) return rc;
    if (int rc = alloc_level<T>(sc, c, dim, N / 2, false, false, false)) return rc;
    if (int rc = load_dense<T>(sc, f.L, u, f.x[0], s)) return rc;
    if (int rc = load_dense<T>(sc, f.L, b, f.b, s)) return rc;
    CK(launch_residual_restrict<T>(f.L, c.L, f.x[0], f.b, c.x[0], f.sA, s));
    return store_dense<T>(sc, c.L, c.x[0], coarse, s);
}

extern "C" int spaimg_residual_restrict(int dtype, int dim, int N, const void* u, const void* b, void* coarse,
                                        void* stream) {
    if (int rc = check_dims(dtype, dim, N)) return rc;
    if (int rc = check_halving(N)) return rc;
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SPAIMG_F64 ? residual_restrict_t<double>(dim, N, u, b, coarse, s)
                               : residual_restrict_t<float>(dim, N, u, b, coarse, s);
}

template <class T>
static int norm_t(int dim, int N, const void* u, const void* b, double* out, cudaStream_t s) {
    Scratch sc(s);
    Level<T> f;
    if (int rc = alloc_level<T>(sc, f, dim, N, false, true, false)) return rc;
    if (int rc = load_dense<T>(sc, f.L, u, f.x[0], s)) return rc;
    if (int rc = load_dense<T>(sc, f.L, b, f.b, s)) return rc;
    double* part = nullptr;
    double* nrm = nullptr;
    unsigned* cnt = nullptr;
    CK(sc.get(&part, kNormBlocks));
    CK(sc.get(&nrm, 1));
    CK(sc.get(&cnt, 1));
    CK(launch_residual_norm<T>(f.L, f.x[0], f.b, f.sA, part, cnt, nrm, 0, nullptr, s));
    CK(cudaMemcpyAsync(out, nrm, sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return 0;
}

extern "C" int spaimg_residual_norm(int dtype, int dim, int N, const void* u, const void* b, double* out, void* stream) {
    if (int rc = check_dims(dtype, dim, N)) return rc;
    if (!out) return fail(SPAIMG_EINVAL, "out is NULL");
    cudaStream_t s = (cudaStream_t)stream;
    return dtype == SPAIMG_F64 ? norm_t<double>(dim, N, u, b, out, s) : norm_t<float>(dim, N, u, b, out, s);
}

// ------------------------------------------------------------------------------------------
// the solver: level hierarchy + captured cycle
// ------------------------------------------------------------------------------------------
struct spaimg_solver {
    virtual ~spaimg_solver() = default;
    virtual int load(const void* b, const void* u0, cudaStream_t s) = 0;
    virtual int cycles(int n, cudaStream_t s) = 0;
    virtual int run(double tol, int max_iters, double* norms, int* iters, int* conv, cudaStream_t s) = 0;
    virtual int store(void* out, cudaStream_t s) = 0;
    virtual int solve_batch(int nrhs, const void* const* b, void* const* u, double tol, int max_iters, double* norms,
                            int* iters, int* conv, cudaStream_t s) = 0;
    virtual int op(int which, int reps, cudaStream_t s) = 0;
    virtual void stats(spaimg_solver_stats* st) const = 0;
};

// ------------------------------------------------------------------------------------------
// device-side solve loop (reference multigrid.py:206-217) as a CUDA graph with a conditional
// WHILE node:   reset -> A -> WHILE(cont) { B -> A }
// A = the norm of u_k fused into cycle k+1's first pre-sweep (which only writes the other
// buffer, so it is harmlessly speculative after the last cycle); the norm kernel's last CTA
// runs the stop test (‖r_k‖ <= tol ‖r_0‖ or k == max_iters) and sets the WHILE condition.
// B = the rest of cycle k+1.  No host round trip per cycle; the history stays on the device.
// ------------------------------------------------------------------------------------------

__global__ void k_solve_reset(int* slot, int* state) {
    *slot = 0;
    state[0] = 0;
    state[1] = 0;
}

template <class T> struct Solver final : spaimg_solver {
    spaimg_mg_config cfg{};
    std::vector<double> lu_h;
    std::vector<int> piv_h;
    std::vector<Level<T>> lv;  // lv[0] finest ... lv.back() = coarse-solve level
    Terms<T> M{};
    int shape = SHAPE_GENERIC;
    bool fused = false;      // fused K1 sweep available for this smoother
    bool fused_norm = false; // norm folded into the first pre-sweep (A) of the next cycle
    T omega{};
    T* lu = nullptr;
    int* piv = nullptr;
    int nlu = 0;
    double* norms_d = nullptr;
    int norms_cap = 0;
    int* slot_d = nullptr;
    int* state_d = nullptr;
    SolveCtl* ctl_d = nullptr;
    double* partials = nullptr;
    unsigned* counter = nullptr;
    double* norms_h = nullptr;  // pinned
    int* state_h = nullptr;     // pinned
    SolveCtl* ctl_h = nullptr;  // pinned
    T* stage = nullptr;         // dense staging on device
    cudaGraphExec_t exec_cycle = nullptr, exec_solve = nullptr;
    int kernels_per_cycle = 0;
    int kernels_a = 0;
    bool use_graph = true;
    std::vector<void*> owned;
    std::vector<std::pair<long long, cudaGraphExec_t>> op_graphs;
    // shared-memory coarse engine (K5+): levels >= tail_l (if < nsmooth()) run in one CTA per visit
    int tail_l = 1 << 30;
    TailArgs<T> tail_args[2] = {};  // complete launch parameters for an entry from a given iterate / from zero
    T* tail_coarse = nullptr;       // coarse factors for nlu > kTailMaxLU
    int* tail_coarse_idx = nullptr;

    ~Solver() override {
        if (bs_h2d) {
            cudaStreamSynchronize(bs_h2d);
            cudaStreamSynchronize(bs_d2h);
            cudaStreamDestroy(bs_h2d);
            cudaStreamDestroy(bs_d2h);
            for (int i = 0; i < 2; ++i) {
                cudaEventDestroy(ev_in[i]);
                cudaEventDestroy(ev_pad[i]);
                cudaEventDestroy(ev_unpad[i]);
                cudaEventDestroy(ev_out[i]);
            }
            cudaEventDestroy(ev_go);
        }
        if (bnorms_h) cudaFreeHost(bnorms_h);
        if (exec_cycle) cudaGraphExecDestroy(exec_cycle);
        if (exec_solve) cudaGraphExecDestroy(exec_solve);
        for (auto& kv : op_graphs) cudaGraphExecDestroy(kv.second);
        for (void* p : owned) cudaFree(p);
        if (norms_h) cudaFreeHost(norms_h);
        if (state_h) cudaFreeHost(state_h);
    }

    template <class U> int dalloc(U** p, size_t count) {
        void* q = nullptr;
        const size_t bytes = count * sizeof(U) > 0 ? count * sizeof(U) : 16;
        CK(cudaMalloc(&q, bytes));
        owned.push_back(q);
        CK(cudaMemset(q, 0, bytes));
        *p = static_cast<U*>(q);
        return 0;
    }

    NormOut norm_sink() const { return NormOut{partials, counter, norms_d, slot_d, nullptr, nullptr, 0}; }
    // the norm sink that also evaluates the stop test and drives the WHILE node (solve graph)
    NormOut norm_sink_cond(cudaGraphConditionalHandle h) const {
        return NormOut{partials, counter, norms_d, slot_d, ctl_d, state_d, h};
    }
    cudaGraphConditionalHandle cur_cond = 0;  // set while capturing the solve graph
    bool in_solve_graph = false;

    int init(const spaimg_mg_config& c) {
        {   // the direct solve keeps the coarse vector in one CTA's shared memory (k_coarse_solve)
            int dev = 0, optin = 0;
            CK(cudaGetDevice(&dev));
            CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
            if ((size_t)c.coarse_n * sizeof(T) > (size_t)optin)
                return fail(SPAIMG_ENOTSUP, "coarse system of " + std::to_string(c.coarse_n) + " unknowns exceeds the direct solve's limit of " +
                                                std::to_string(optin / (int)sizeof(T)) + " (choose a smaller coarsest_N)");
        }
        cfg = c;
        lu_h.assign(c.coarse_lu, c.coarse_lu + (size_t)c.coarse_n * c.coarse_n);
        piv_h.assign(c.coarse_piv, c.coarse_piv + c.coarse_n);
        cfg.coarse_lu = nullptr;
        cfg.coarse_piv = nullptr;
        const char* eg = getenv("SPAIMG_NO_GRAPH");
        use_graph = !(eg && eg[0] == '1');
        M = to_terms<T>(c.M);
        shape = detect_shape(c.M);
        fused = stencil_radius(c.M) <= 1 && sweep_fused_supported(c.dim, shape);
        omega = (T)c.omega;
        // levels: halve until N <= coarsest_N (multigrid.py:166, :178); the zero frame is as wide
        // as the smoother's reach (stencils.py:139-146), at least the kernels' two cells
        const int ghost = std::max(kGhost, stencil_radius(c.M));
        int N = c.N;
        while (true) {
            Level<T> l;
            l.L = make_layout(c.dim, N, sizeof(T), ghost);
            l.sA = (T)hscale(N, -2);
            l.sM = (T)hscale(N, c.M.h_exponent);
            const bool coarse = N <= c.coarsest_N;
            if (int rc = dalloc(&l.x[0], (size_t)l.L.alloc)) return rc;
            if (int rc = dalloc(&l.b, (size_t)l.L.alloc)) return rc;
            if (!coarse) {
                if (int rc = dalloc(&l.x[1], (size_t)l.L.alloc)) return rc;
                if (!fused)  // the unfused residual + relax sweep (stencil radius >= 2)
                    if (int rc = dalloc(&l.r, (size_t)l.L.alloc)) return rc;
            }
            if constexpr (kDebugChecks) {
                for (T* buf : {l.x[0], l.x[1], l.b, l.r})
                    if (buf) CK(launch_poison_level<T>(l.L, buf, 0));
            }
            lv.push_back(l);
            if (coarse) break;
            if (N % 2) return fail(SPAIMG_EINVAL, "cannot halve an odd mesh count N=" + std::to_string(N));
            if (N / 2 < 2) return fail(SPAIMG_EINVAL, "coarse mesh would have no interior points");
            N /= 2;
        }
        if (N != c.coarse_N || count_of(c.dim, N) != c.coarse_n)
            return fail(SPAIMG_EINVAL, "coarse factorisation does not match the coarsest level");
        fused_norm = nsmooth() >= 1 && c.nu1 >= 1 && fused;
        const char* e2 = getenv("SPAIMG_SWEEP2");
        pair_sweeps = !(e2 && e2[0] == '0');
        plan_solve = make_plan(true);
        plan_cycle = make_plan(false);
        nlu = c.coarse_n;
        std::vector<T> luT(lu_h.begin(), lu_h.end());
        if (int rc = dalloc(&lu, luT.size())) return rc;
        CK(cudaMemcpy(lu, luT.data(), luT.size() * sizeof(T), cudaMemcpyHostToDevice));
        if (int rc = dalloc(&piv, piv_h.size())) return rc;
        CK(cudaMemcpy(piv, piv_h.data(), piv_h.size() * sizeof(int), cudaMemcpyHostToDevice));
        if (int rc = init_tail()) return rc;
        norms_cap = 0;
        if (int rc = grow_norms(101)) return rc;  // the reference default max_iters = 100; grown on demand
        if (int rc = dalloc(&slot_d, 1)) return rc;
        if (int rc = dalloc(&state_d, 2)) return rc;
        if (int rc = dalloc(&ctl_d, 1)) return rc;
        if (int rc = dalloc(&partials, 1 << 16)) return rc;
        if (int rc = dalloc(&counter, 1)) return rc;
        if (int rc = dalloc(&stage, (size_t)count_of(c.dim, c.N))) return rc;
        void* ph = nullptr;
        CK(cudaMallocHost(&ph, 64 + sizeof(SolveCtl)));
        state_h = static_cast<int*>(ph);
        ctl_h = reinterpret_cast<SolveCtl*>(static_cast<char*>(ph) + 64);
        // every buffer above was zeroed on the legacy stream; the solver runs on the caller's
        // (possibly non-blocking) stream, so finish that work before returning
        CK(cudaDeviceSynchronize());
        return 0;
    }

    // residual-history buffers for at least `cap` norms (device + pinned host).  The graphs read
    // norms_d through NormOut by value, so growing re-captures them.
    int grow_norms(int cap) {
        if (cap <= norms_cap) return 0;
        double* d = nullptr;
        CK(cudaMalloc(&d, sizeof(double) * cap));
        CK(cudaMemset(d, 0, sizeof(double) * cap));
        double* h = nullptr;
        CK(cudaMallocHost(&h, sizeof(double) * cap));
        if (norms_d) {
            CK(cudaMemcpy(d, norms_d, sizeof(double) * norms_cap, cudaMemcpyDeviceToDevice));
            cudaFree(norms_d);
            owned.erase(std::remove(owned.begin(), owned.end(), (void*)norms_d), owned.end());
        }
        if (norms_h) cudaFreeHost(norms_h);
        norms_d = d;
        norms_h = h;
        owned.push_back(d);
        norms_cap = cap;
        if (exec_cycle) cudaGraphExecDestroy(exec_cycle);
        if (exec_solve) cudaGraphExecDestroy(exec_solve);
        exec_cycle = exec_solve = nullptr;
        for (auto& kv : op_graphs) cudaGraphExecDestroy(kv.second);
        op_graphs.clear();
        return 0;
    }

    int nsmooth() const { return (int)lv.size() - 1; }

    // largest mesh count run by the shared-memory engine (SPAIMG_TAIL_N overrides; 0 disables).
    // The engine maps a level onto a box of at most 64^2 / 16^3 points.
    static int tail_threshold(const spaimg_mg_config& c) {
        const char* e = getenv("SPAIMG_TAIL_N");
        if (e) return atoi(e);
        return c.dim == 2 ? 64 : 16;
    }

    // ---- shared-memory engine plan ------------------------------------------------------
    struct HOp {
        int type, level, nw, bw, bid;
    };
    std::vector<TailLv<T>> tg;  // tail levels: tg[0] = entry level ... tg.back() = coarse level

    static int ceil_log2(int n) {
        int k = 0;
        while ((1 << k) < n) ++k;
        return k;
    }
    static int warps_for(int dim, int logw) {
        const long long pts = 1LL << (dim * logw);
        const long long act = pts > kTailThreads ? kTailThreads : pts;
        return (int)((act + 31) / 32);
    }

    // levels l0 .. nsmooth() in shared memory: geometry; returns the array block size (elements)
    int plan_geometry(int l0, int F, int* zero_from) {
        tg.clear();
        int cur = 0;
        for (int l = l0; l <= nsmooth(); ++l) {
            TailLv<T> g{};
            g.n = lv[l].L.n;
            g.logw = ceil_log2(g.n);
            const int w = g.n + 2 * F;
            g.s0 = cfg.dim == 2 ? w : w * w;
            g.s1 = cfg.dim == 3 ? w : 0;
            const int size = ((cfg.dim == 2 ? w * w : w * w * w) + 1) / 2 * 2;  // 16-byte multiples
            const int origin = F * g.s0 + F * g.s1 + F;
            g.x = cur + origin;
            cur += size;
            g.b = cur + origin;
            cur += size;
            if (l == l0) *zero_from = cur;
            if (l < nsmooth()) {
                g.r = cur + origin;
                cur += size;
            } else {
                g.r = -1;
            }
            g.sA = lv[l].sA;
            g.sM = lv[l].sM;
            tg.push_back(g);
        }
        // strips may read up to two axis-0 rows past an array (values unused): keep them in bounds
        return cur + 2 * tg[0].s0 + 2 * tg[0].s1 + 2;
    }

    HOp point_op(int type, int i) const {
        const int logw = type == TAIL_FW ? tg[i].logw - 1 : tg[i].logw;
        return HOp{type, i, warps_for(cfg.dim, logw), 0, 0};
    }

    // the recursion of visit() (multigrid.py:157-185) below the entry level, as engine ops
    void record(int i, bool fz, std::vector<HOp>& ops) const {
        const int last = (int)tg.size() - 1;
        if (i == last) {  // u.N <= coarsest_N: direct solve (multigrid.py:166-167)
            ops.push_back(HOp{TAIL_COARSE, i, nlu <= kTailMaxLU ? 1 : kTailThreads / 32, 0, 0});
            return;
        }
        for (int k = 0; k < cfg.nu1; ++k) {
            if (fz && k == 0) {
                ops.push_back(point_op(TAIL_RELAX0, i));
            } else {
                ops.push_back(point_op(TAIL_RES, i));
                ops.push_back(point_op(TAIL_RELAX, i));
            }
        }
        if (fz && cfg.nu1 == 0) ops.push_back(point_op(TAIL_ZERO, i));
        ops.push_back(point_op(TAIL_RES, i));
        ops.push_back(point_op(TAIL_FW, i));
        record(i + 1, true, ops);
        // the restricted system of the coarsest level is solved once, whatever gamma
        // (multigrid.py:178-179)
        if (i + 1 < last)
            for (int g = 1; g < cfg.gamma; ++g) record(i + 1, false, ops);
        ops.push_back(point_op(TAIL_PROLONG, i));
        for (int k = 0; k < cfg.nu2; ++k) {
            ops.push_back(point_op(TAIL_RES, i));
            ops.push_back(point_op(TAIL_RELAX, i));
        }
    }

    // the op sequence of the compile-time engine (kernels_tail_fast.cuh visit()), for the
    // SPAIMG_TAIL_PROF labels
    // kernels_tail_fast.cuh FastTail::NTH / fuse_rr / fuse_pr
    int fast_nth(int) const { return kTailThreads; }
    bool fast_fuse_rr(int i) const {
        const int lw = tg[i].logw;
        if (i + 1 >= (int)tg.size()) return false;
        return cfg.dim == 2 && (1LL << (cfg.dim * (lw - 1))) <= fast_nth(i + 1);
    }
    void record_fast(int i, bool fz, std::vector<HOp>& ops) const {
        const int last = (int)tg.size() - 1;
        for (int k = 0; k < cfg.nu1; ++k) {
            if (fz && k == 0) {
                ops.push_back(point_op(TAIL_RELAX0, i));
            } else {
                ops.push_back(point_op(TAIL_RES, i));
                ops.push_back(point_op(TAIL_RELAX, i));
            }
        }
        if (fz && cfg.nu1 == 0) ops.push_back(point_op(TAIL_ZERO, i));
        if (fast_fuse_rr(i)) {
            HOp o = point_op(TAIL_FW, i);
            o.type = TAIL_RESFW;
            ops.push_back(o);
        } else {
            ops.push_back(point_op(TAIL_RES, i));
            ops.push_back(point_op(TAIL_FW, i));
        }
        if (i + 1 == last) {
            ops.push_back(HOp{TAIL_COARSE, last, 1, 0, 0});
        } else {
            for (int g = 0; g < cfg.gamma; ++g) record_fast(i + 1, g == 0, ops);
        }
        ops.push_back(point_op(TAIL_PROLONG, i));
        for (int k = 0; k < cfg.nu2; ++k) {
            ops.push_back(point_op(TAIL_RES, i));
            ops.push_back(point_op(TAIL_RELAX, i));
        }
    }

    // barrier plan: op i waits with the warps of ops i-1 and i (always a prefix of the CTA); one
    // named barrier id per distinct warp count -- warps that skip small ops run ahead and must
    // not share a barrier with a different count
    int tail_barriers(std::vector<HOp>& ops) const {
        std::vector<int> counts;
        const int all = kTailThreads / 32;
        int prev = all;
        for (HOp& o : ops) {
            o.bw = std::max(o.nw, prev);
            prev = o.nw;
            if (o.bw == all) {
                o.bid = 0;
            } else if (o.bw == 1) {
                o.bid = kTailSyncWarp;
            } else {
                auto it = std::find(counts.begin(), counts.end(), o.bw);
                if (it == counts.end()) {
                    counts.push_back(o.bw);
                    it = counts.end() - 1;
                }
                o.bid = (int)(it - counts.begin()) + 1;
            }
        }
        if (counts.size() > 15) return fail(SPAIMG_ENOTSUP, "tail: too many distinct warp counts for named barriers");
        return 0;
    }

    int init_tail() {
        const int thr = tail_threshold(cfg);
        if (thr <= 0) return 0;
        const int F = std::max(1, stencil_radius(cfg.M));
        if (F > lv[0].L.ghost) return 0;
        const int nmax = cfg.dim == 2 ? 63 : 15;  // the engine's largest W^dim box
        int dev = 0, optin = 0;
        CK(cudaGetDevice(&dev));
        CK(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
        int l0 = nsmooth();
        while (l0 > 1 && lv[l0 - 1].L.N <= thr && lv[l0 - 1].L.n <= nmax) --l0;  // the finest level never joins
        if (l0 >= nsmooth()) return 0;
        // shrink the engine until its levels fit in one CTA's shared memory and its op lists in
        // the launch parameters
        std::vector<HOp> ops[2];
        int arr_elems = 0, zero_from = 0;
        size_t smem = 0;
        for (; l0 < nsmooth(); ++l0) {
            if (nsmooth() + 1 - l0 > kTailMaxLevels) continue;
            arr_elems = plan_geometry(l0, F, &zero_from);
            for (int fz = 0; fz < 2; ++fz) {
                ops[fz].clear();
                record(0, fz != 0, ops[fz]);
                if (int rc = tail_barriers(ops[fz])) return rc;
            }
            if ((int)std::max(ops[0].size(), ops[1].size()) > kTailMaxOps) continue;
            smem = ((size_t)arr_elems + (nlu > kTailMaxLU ? (size_t)nlu * nlu + 3 * (size_t)nlu + 2 : 0)) * sizeof(T) +
                   (nlu > kTailMaxLU ? (2 * (size_t)nlu + 2) * sizeof(int) : 0);
            if (smem <= (size_t)optin) break;
        }
        if (l0 >= nsmooth()) return 0;
        tail_l = l0;
        // coarse data: -LU off the diagonal, U_jj, 1/U_jj (correctly rounded host division);
        // the row interchanges of getrs (laswp) folded into a gather order
        std::vector<T> cf((size_t)nlu * nlu + 2 * (size_t)nlu);
        for (int i = 0; i < nlu; ++i)
            for (int j = 0; j < nlu; ++j) cf[(size_t)i * nlu + j] = i == j ? T(0) : (T)(-lu_h[(size_t)i * nlu + j]);
        for (int j = 0; j < nlu; ++j) {
            const T d = (T)lu_h[(size_t)j * nlu + j];
            cf[(size_t)nlu * nlu + j] = d;
            cf[(size_t)nlu * nlu + nlu + j] = T(1) / d;
        }
        std::vector<int> perm(nlu), ci(2 * (size_t)nlu);
        for (int i = 0; i < nlu; ++i) perm[i] = i;
        for (int i = 0; i < nlu; ++i) std::swap(perm[i], perm[piv_h[i]]);
        const TailLv<T>& cg = tg.back();
        auto off = [&](int q) {
            const int n = cg.n;
            if (cfg.dim == 2) return (q / n) * cg.s0 + q % n;
            return (q / (n * n)) * cg.s0 + ((q / n) % n) * cg.s1 + q % n;
        };
        for (int i = 0; i < nlu; ++i) {
            ci[i] = off(perm[i]);
            ci[nlu + i] = off(i);
        }
        if (nlu > kTailMaxLU) {
            if (int rc = dalloc(&tail_coarse, cf.size())) return rc;
            CK(cudaMemcpy(tail_coarse, cf.data(), cf.size() * sizeof(T), cudaMemcpyHostToDevice));
            if (int rc = dalloc(&tail_coarse_idx, ci.size())) return rc;
            CK(cudaMemcpy(tail_coarse_idx, ci.data(), ci.size() * sizeof(int), cudaMemcpyHostToDevice));
        }
        long long* prof = nullptr;
        const char* ep = getenv("SPAIMG_TAIL_PROF");
        if (ep && ep[0] == '1')
            if (int rc = dalloc(&prof, (size_t)3 * kTailMaxOps + 1)) return rc;
        // the compile-time engine: a power-of-two hierarchy from the instantiated entry size down to
        // a coarse level of 1 or 3 points per axis, frame 1, a named smoother shape
        const int le = cfg.dim == 2 ? kTailFastLE2 : kTailFastLE3;
        bool fast = F == 1 && tail_fast_shape(cfg.dim, shape) && tg[0].n == (1 << le) - 1;
        for (size_t i = 0; i < tg.size(); ++i) fast = fast && tg[i].n == (1 << (le - (int)i)) - 1;
        const int lc = le - (int)tg.size() + 1;
        fast = fast && (lc == 1 || lc == 2);
        const char* ef = getenv("SPAIMG_TAIL_FAST");
        if (ef && ef[0] == '0') fast = false;
        for (int fz = 0; fz < 2; ++fz) {
            TailArgs<T>& ta = tail_args[fz];
            ta.gamma = cfg.gamma;
            ta.nu1 = cfg.nu1;
            ta.nu2 = cfg.nu2;
            ta.entry_fz = fz;
            ta.fast_le = fast ? le : 0;
            ta.fast_lc = fast ? lc : 0;
            ta.nops = (int)ops[fz].size();
            ta.nlv = (int)tg.size();
            ta.nlu = nlu;
            ta.arr_elems = arr_elems;
            ta.zero_from = zero_from;
            ta.frame = F;
            ta.smem = smem;
            ta.M = M;
            ta.omega = omega;
            ta.gL = lv[l0].L;
            ta.shape = shape;
            ta.prof = prof;
            ta.coarse_g = tail_coarse;
            ta.coarse_idx_g = tail_coarse_idx;
            for (size_t i = 0; i < tg.size(); ++i) ta.lv[i] = tg[i];
            if (nlu <= kTailMaxLU) {
                for (int i = 0; i < nlu; ++i)
                    for (int j = 0; j < nlu; ++j) ta.lu[i * nlu + j] = cf[(size_t)i * nlu + j];
                for (int j = 0; j < nlu; ++j) {
                    ta.dg[j] = cf[(size_t)nlu * nlu + j];
                    ta.rc[j] = cf[(size_t)nlu * nlu + nlu + j];
                    ta.cin[j] = ci[j];
                    ta.cout[j] = ci[nlu + j];
                }
            }
            for (size_t i = 0; i < ops[fz].size(); ++i) {
                const HOp& o = ops[fz][i];
                ta.ops[i] = tail_op_word(o.type, o.level, o.nw, o.bw, o.bid);
            }
        }
        prof_ops[0] = ops[0];
        prof_ops[1] = ops[1];
        if (fast)
            for (int fz = 0; fz < 2; ++fz) {
                prof_ops[fz].clear();
                record_fast(0, fz != 0, prof_ops[fz]);
            }
        return 0;
    }

    // diagnostics: per-op cycles of the last engine launch (SPAIMG_TAIL_PROF=1, eager runs)
    std::vector<HOp> prof_ops[2];
    int prof_last_fz = 0;
    void tail_profile_dump() {
        if (!tail_args[0].prof) return;
        const std::vector<HOp>& ops = prof_ops[prof_last_fz];
        std::vector<long long> c(3 * kTailMaxOps + 1);
        if (cudaDeviceSynchronize() != cudaSuccess) return;
        cudaMemcpy(c.data(), tail_args[0].prof, c.size() * sizeof(long long), cudaMemcpyDeviceToHost);
        c[ops.size()] = c[ops.size()];
        static const char* names[] = {"RES", "RELAX", "RELAX0", "ZERO", "FW", "PROLONG", "COARSE", "RESFW"};
        long long tot[8] = {}, cnt[8] = {};
        for (size_t i = 0; i < ops.size(); ++i) {
            const long long d = c[i + 1] - c[i];
            tot[ops[i].type] += d;
            cnt[ops[i].type] += 1;
            const bool split = ops[i].type != TAIL_COARSE && !tail_args[0].fast_le;
            const long long pre = split ? c[kTailMaxOps + i] - c[i] : 0;
            const long long body = split ? c[2 * kTailMaxOps + i] - c[kTailMaxOps + i] : 0;
            fprintf(stderr, "tailprof op %3zu %-7s n=%2d nw=%2d bw=%2d  %6lld cycles (dispatch %lld body %lld)\n", i,
                    names[ops[i].type], tg[ops[i].level].n, ops[i].nw, ops[i].bw, d, pre, body);
        }
        for (int k = 0; k < 8; ++k)
            if (cnt[k]) fprintf(stderr, "tailprof sum %-7s %3lld ops %8lld cycles\n", names[k], cnt[k], tot[k]);
        fprintf(stderr, "tailprof total %lld cycles\n", c[ops.size()] - c[0]);
        if (tail_args[0].fast_le)
            fprintf(stderr, "tailprof entry -> first op %lld cycles, last op -> exit %lld cycles\n",
                    c[0] - c[2 * kTailMaxOps], c[2 * kTailMaxOps + 1] - c[ops.size()]);
    }

    // one visit of the engine's entry level: x[a] updated in place
    int tail_visit(int l, int a, bool fz, cudaStream_t s, int* launches) {
        if (l != tail_l) return -1;
        const int z = fz ? 1 : 0;
        TailArgs<T>& ta = tail_args[z];
        ta.gb = lv[l].b;
        ta.gx = lv[l].x[a];
        prof_last_fz = z;
        if (launch_tail<T>(ta, s) != cudaSuccess) return -1;
        ++*launches;
        return a;
    }

    // ||b - A x||_2 of the finest level appended to the device history
    int norm_launch(const T* x, cudaStream_t s, int* launches) {
        const Level<T>& L = lv[0];
        CK(launch_norm_march<T>(L.L, x, L.b, L.sA, in_solve_graph ? norm_sink_cond(cur_cond) : norm_sink(), s));
        ++*launches;
        return 0;
    }

    // ---- pairing smoothing steps into two-sweep marches (launch_sweep2) ---------------------
    // A pass is one launch writing the other x buffer: one sweep, or two sweeps in one march on
    // the 2D marching levels (24 B/unknown per pair instead of 48).  Levels >= 1 pair greedily
    // (visit() returns whichever buffer its result lands in).  Level 0 must end a cycle in x[0]:
    // its plan picks the most pairs whose pass count is even (a prolongation not fused into a
    // sweep can also flip, writing the other buffer).
    struct Level0Plan {
        int a_sweeps = 0;    // sweeps done by part A (0: no part A in this schedule)
        int pre_pairs = 0;   // pairs among the remaining pre-sweeps
        int post_pairs = 0;  // pairs among the post-sweeps (the first one carries the K3 when fused)
        bool pc = false;     // K3 fused into the first post pass
        bool k3_flip = false;  // unfused K3 writes the other buffer
    };
    Level0Plan plan_solve, plan_cycle;
    const Level0Plan* plan0 = &plan_cycle;

    bool pair_sweeps = true;  // SPAIMG_SWEEP2=0: one sweep per launch everywhere (comparison knob)
    bool two_ok(int l) const { return pair_sweeps && fused && sweep2_supported(lv[l].L, shape); }

    Level0Plan make_plan(bool with_a) const {
        const int nu1 = cfg.nu1, nu2 = cfg.nu2;
        const bool two0 = nsmooth() >= 1 && two_ok(0);
        const bool pc_ok = nsmooth() >= 1 && nu2 >= 1 && fused && sweep_pc_supported(lv[0].L, shape);
        const bool has_a = with_a && fused_norm;
        Level0Plan best;
        int best_pairs = -1;
        for (int a2 = (has_a && two0 && nu1 >= 2) ? 1 : 0; a2 >= 0; --a2) {
            const int a_sw = has_a ? 1 + a2 : 0;
            const int r1 = nu1 - a_sw;
            for (int pp = two0 ? r1 / 2 : 0; pp >= 0; --pp)
                for (int pc = pc_ok ? 1 : 0; pc >= 0; --pc)
                    for (int qq = two0 ? nu2 / 2 : 0; qq >= 0; --qq) {
                        const int passes = (has_a ? 1 : 0) + (r1 - pp) + (nu2 - qq);
                        const bool flip = !pc && (passes & 1);  // an unfused K3 can fix the parity
                        if (pc && (passes & 1)) continue;
                        const int pairs = a2 + pp + qq + (pc ? 1 : 0);
                        if (pairs > best_pairs) {
                            best_pairs = pairs;
                            best.a_sweeps = a_sw;
                            best.pre_pairs = pp;
                            best.post_pairs = qq;
                            best.pc = pc != 0;
                            best.k3_flip = flip;
                        }
                    }
        }
        return best;
    }

    // one pass of `two ? 2 : 1` sweeps on level l: x[a] -> x[1-a]
    int sweep_pass(int l, int a, bool fz, bool two, cudaStream_t s, int* launches) {
        Level<T>& L = lv[l];
        if (two) {
            if (launch_sweep2<T>(L.L, L.x[a], L.b, L.x[1 - a], M, shape, L.sA, L.sM, omega, fz, s) != cudaSuccess)
                return -1;
            ++*launches;
            return 0;
        }
        return do_sweep<T>(L, a, fz, M, shape, fused, omega, s, launches) ? -1 : 0;
    }

    // recursive schedule (multigrid.py:157-185).  Returns the buffer index of level l holding
    // the result, or -1 on error.  a: the buffer holding the start iterate after the pre_done
    // pre-sweeps already applied (level 0: part A; small 2D levels: the finer level's residual +
    // restriction kernel carries the coarse level's first, zero-start sweep).
    int visit(int l, int a, bool fz, cudaStream_t s, int* launches, int pre_done) {
        if (l >= tail_l && l < nsmooth()) return tail_visit(l, a, fz, s, launches);
        Level<T>& L = lv[l];
        if (l == nsmooth()) {  // u.N <= coarsest_N: direct solve (multigrid.py:166-167)
            if (launch_coarse_solve<T>(L.L, L.b, L.x[0], lu, piv, nlu, s) != cudaSuccess) return -1;
            ++*launches;
            return 0;
        }
        const bool two = two_ok(l);
        int pairs = l == 0 ? plan0->pre_pairs : (two ? 1 << 20 : 0);
        for (int k = pre_done; k < cfg.nu1;) {
            const bool pair = two && pairs > 0 && cfg.nu1 - k >= 2;
            if (sweep_pass(l, a, fz, pair, s, launches)) return -1;
            k += pair ? 2 : 1;
            pairs -= pair ? 1 : 0;
            a = 1 - a;
            fz = false;
        }
        if (fz) {  // nu1 == 0 on a zero start: materialise the zero iterate
            if (cudaMemsetAsync(L.x[a], 0, (size_t)L.L.alloc * sizeof(T), s) != cudaSuccess) return -1;
            ++*launches;
        }
        Level<T>& C = lv[l + 1];
        // on the small 2D levels the coarse level's first (zero-start) pre-sweep rides with K2
        // (measured: c2 -1.7 %, c1 -3.5 %; in 3D the ring recomputation costs more than the
        // launch it saves, c3 +7 %, so 3D keeps two kernels)
        const bool rr_fz = fused && cfg.nu1 >= 1 && l + 1 < nsmooth() && l + 1 < tail_l &&
                           L.L.N <= flat_threshold(cfg.dim) && cfg.dim == 2;
        if (rr_fz) {
            if (launch_residual_restrict_fz<T>(L.L, C.L, L.x[a], L.b, C.b, C.x[1], M, shape, L.sA, C.sM, omega, s) !=
                cudaSuccess)
                return -1;
        } else {
            if (launch_residual_restrict<T>(L.L, C.L, L.x[a], L.b, C.b, L.sA, s) != cudaSuccess) return -1;
        }
        ++*launches;
        int c;
        if (l + 1 == nsmooth()) {
            if (launch_coarse_solve<T>(C.L, C.b, C.x[0], lu, piv, nlu, s) != cudaSuccess) return -1;
            ++*launches;
            c = 0;
        } else {
            c = visit(l + 1, rr_fz ? 1 : 0, !rr_fz, s, launches, rr_fz ? 1 : 0);
            for (int g = 1; g < cfg.gamma && c >= 0; ++g) c = visit(l + 1, c, false, s, launches, 0);
            if (c < 0) return -1;
        }
        // post-smoothing; the prolongation + correction (multigrid.py:184) fused into the first
        // post pass where the level allows it
        int ppairs = l == 0 ? plan0->post_pairs : (two ? 1 << 20 : 0);
        const bool pc = l == 0 ? plan0->pc : (cfg.nu2 >= 1 && fused && sweep_pc_supported(L.L, shape));
        int k = 0;
        if (pc) {
            const bool pair = two && ppairs > 0 && cfg.nu2 >= 2;
            const cudaError_t e =
                pair ? launch_sweep2_pc<T>(L.L, C.L, L.x[a], C.x[c], L.b, L.x[1 - a], M, shape, L.sA, L.sM, omega, s)
                     : launch_sweep_pc<T>(L.L, C.L, L.x[a], C.x[c], L.b, L.x[1 - a], M, shape, L.sA, L.sM, omega, s);
            if (e != cudaSuccess) return -1;
            ++*launches;
            a = 1 - a;
            k = pair ? 2 : 1;
            ppairs -= pair ? 1 : 0;
        } else {
            const int ao = (l == 0 && plan0->k3_flip) ? 1 - a : a;
            if (launch_prolong_correct<T>(L.L, C.L, L.x[a], L.x[ao], C.x[c], s) != cudaSuccess) return -1;
            ++*launches;
            a = ao;
        }
        while (k < cfg.nu2) {
            const bool pair = two && ppairs > 0 && cfg.nu2 - k >= 2;
            if (sweep_pass(l, a, false, pair, s, launches)) return -1;
            k += pair ? 2 : 1;
            ppairs -= pair ? 1 : 0;
            a = 1 - a;
        }
        return a;
    }

    // A: norm of the iterate in x[0] (+ the first pre-sweep(s) of the next cycle when fused)
    int part_a(cudaStream_t s, int* launches) {
        if (fused_norm) {
            Level<T>& L = lv[0];
            const NormOut no = in_solve_graph ? norm_sink_cond(cur_cond) : norm_sink();
            if (plan_solve.a_sweeps == 2)
                CK(launch_sweep2<T>(L.L, L.x[0], L.b, L.x[1], M, shape, L.sA, L.sM, omega, false, s, &no));
            else
                CK(launch_sweep<T>(L.L, L.x[0], L.b, L.x[1], M, shape, L.sA, L.sM, omega, false, s, &no));
            ++*launches;
            return 0;
        }
        return norm_launch(lv[0].x[0], s, launches);
    }

    // B: the rest of the cycle; ends with the iterate back in x[0]
    int part_b(cudaStream_t s, int* launches) {
        plan0 = &plan_solve;
        const int out = visit(0, fused_norm ? 1 : 0, false, s, launches, plan_solve.a_sweeps);
        plan0 = &plan_cycle;
        if (out != 0) return fail(SPAIMG_EINVAL, out < 0 ? "cycle launch failed: " + g_err : "cycle parity error");
        return 0;
    }

    template <class F> int capture_into(cudaGraph_t g, F&& body) {
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        cudaError_t e = cudaStreamBeginCaptureToGraph(cs, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
        if (e != cudaSuccess) {
            cudaStreamDestroy(cs);
            return fail((int)e, std::string("begin capture: ") + cudaGetErrorString(e));
        }
        const int rc = body(cs);
        cudaGraph_t out;
        e = cudaStreamEndCapture(cs, &out);
        cudaStreamDestroy(cs);
        if (rc) return rc;
        if (e != cudaSuccess) return fail((int)e, std::string("end capture: ") + cudaGetErrorString(e));
        return 0;
    }

    // add a conditional node after the current capture dependencies of cs; returns its body
    int add_conditional(cudaStream_t cs, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                        cudaGraph_t* body) {
        cudaStreamCaptureStatus st;
        cudaGraph_t cg;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        CK(cudaStreamGetCaptureInfo(cs, &st, nullptr, &cg, &deps, &nd));
        cudaGraphNodeParams p{};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = type;
        p.conditional.size = 1;
        cudaGraphNode_t node;
        CK(cudaGraphAddNode(&node, cg, deps, nd, &p));
        CK(cudaStreamUpdateCaptureDependencies(cs, &node, 1, cudaStreamSetCaptureDependencies));
        *body = p.conditional.phGraph_out[0];
        return 0;
    }

    // reset; A; WHILE(cont) { B; A }  (see the comment above k_solve_reset)
    int build_solve_graph() {
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        int launches_a = 0, launches_b = 0, dummy = 0;
        cudaGraphConditionalHandle hw;
        cudaGraph_t wbody = nullptr;
        int rc = 0;
        cudaError_t e = cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault);
        if (e != cudaSuccess) rc = fail((int)e, "conditional handle");
        in_solve_graph = true;
        cur_cond = hw;
        if (!rc)
            rc = capture_into(g, [&](cudaStream_t cs) -> int {
                CK(launch_k(k_solve_reset, dim3(1), dim3(1), 0, cs, slot_d, state_d));
                if (int r = part_a(cs, &dummy)) return r;
                return add_conditional(cs, hw, cudaGraphCondTypeWhile, &wbody);
            });
        if (!rc)
            rc = capture_into(wbody, [&](cudaStream_t cs) -> int {
                if (int r = part_b(cs, &launches_b)) return r;
                return part_a(cs, &launches_a);
            });
        in_solve_graph = false;
        if (!rc) {
            e = cudaGraphInstantiate(&exec_solve, g, 0);
            if (e != cudaSuccess) rc = fail((int)e, std::string("solve graph instantiate: ") + cudaGetErrorString(e));
        }
        cudaGraphDestroy(g);
        if (!rc) {
            kernels_per_cycle = launches_a + launches_b;
            kernels_a = launches_a;
        }
        return rc;
    }

    int build_cycle_graph() {
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        int launches = 0;
        int rc = capture_into(g, [&](cudaStream_t cs) -> int {
            const int out = visit(0, 0, false, cs, &launches, 0);
            if (out != 0) return fail(SPAIMG_EINVAL, "cycle capture failed: " + g_err);
            return norm_launch(lv[0].x[0], cs, &launches);
        });
        if (!rc) {
            cudaError_t e = cudaGraphInstantiate(&exec_cycle, g, 0);
            if (e != cudaSuccess) rc = fail((int)e, "cycle graph instantiate");
        }
        cudaGraphDestroy(g);
        return rc;
    }
    int load(const void* b, const void* u0, cudaStream_t s) override {
        Scratch sc(s);
        Level<T>& L = lv[0];
        if (b)  // NULL keeps the right-hand side already loaded
            if (int rc = load_dense<T>(sc, L.L, b, L.b, s, stage)) return rc;
        if (u0) {
            if (int rc = load_dense<T>(sc, L.L, u0, L.x[0], s, stage)) return rc;
        } else {
            CK(cudaMemsetAsync(L.x[0], 0, (size_t)L.L.alloc * sizeof(T), s));
        }
        CK(cudaMemsetAsync(slot_d, 0, sizeof(int), s));
        hist_len = 0;
        return 0;
    }

    // norms appended to the device history since the last reset of its cursor (load / run)
    long long hist_len = 0;

    // n full cycles (each appends its residual norm to the device history, grown as needed)
    int cycles(int n, cudaStream_t s) override {
        if (hist_len + n > (1LL << 24)) return fail(SPAIMG_EINVAL, "too many cycles without a reload");
        if (int rc = grow_norms((int)(hist_len + n))) return rc;
        hist_len += n;
        if (use_graph && !exec_cycle)
            if (int rc = build_cycle_graph()) return rc;
        for (int k = 0; k < n; ++k) {
            if (use_graph) {
                CK(cudaGraphLaunch(exec_cycle, s));
            } else {
                int launches = 0;
                if (visit(0, 0, false, s, &launches, 0) != 0) return fail(SPAIMG_EINVAL, "cycle failed: " + g_err);
                if (int rc = norm_launch(lv[0].x[0], s, &launches)) return rc;
            }
        }
        tail_profile_dump();
        return 0;
    }

    int run(double tol, int max_iters, double* norms, int* iters, int* conv, cudaStream_t s) override {
        if (int rc = grow_norms(max_iters + 1)) return rc;
        hist_len = 0;
        if (!use_graph) return run_host_loop(tol, max_iters, norms, iters, conv, s);
        if (!exec_solve)
            if (int rc = build_solve_graph()) return rc;
        ctl_h->tol = tol;
        ctl_h->max_iters = max_iters;
        CK(cudaMemcpyAsync(ctl_d, ctl_h, sizeof(SolveCtl), cudaMemcpyHostToDevice, s));
        CK(cudaGraphLaunch(exec_solve, s));
        CK(cudaMemcpyAsync(state_h, state_d, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(norms_h, norms_d, sizeof(double) * (max_iters + 1), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        const int k = state_h[0];
        for (int i = 0; i <= k; ++i) norms[i] = norms_h[i];
        *iters = k;
        *conv = state_h[1];
        return 0;
    }

    // eager variant (SPAIMG_NO_GRAPH=1): same schedule, one host round trip per cycle
    int run_host_loop(double tol, int max_iters, double* norms, int* iters, int* conv, cudaStream_t s) {
        CK(cudaMemsetAsync(slot_d, 0, sizeof(int), s));
        int launches = 0, k = 0;
        *conv = 0;
        while (true) {
            if (int rc = part_a(s, &launches)) return rc;
            CK(cudaMemcpyAsync(norms_h + k, norms_d + k, sizeof(double), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            norms[k] = norms_h[k];
            if (k >= 1 && norms[k] <= tol * norms[0]) {
                *conv = 1;
                break;
            }
            if (k >= max_iters) break;
            if (int rc = part_b(s, &launches)) return rc;
            ++k;
        }
        *iters = k;
        return 0;
    }

    int store(void* out, cudaStream_t s) override {
        Scratch sc(s);
        return store_dense<T>(sc, lv[0].L, lv[0].x[0], out, s, stage);
    }

    // ---- pipelined independent solves (host in -> device solve -> host out) -----------------
    // Right-hand side i+1 is copied in (own stream) and solution i-1 copied out (own stream)
    // while solve i runs, through two dense device staging buffers per direction; with pinned
    // host buffers PCIe traffic in both directions overlaps the solves.
    cudaStream_t bs_h2d = nullptr, bs_d2h = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_pad[2] = {}, ev_unpad[2] = {}, ev_out[2] = {}, ev_go = nullptr;
    T* bstage_in[2] = {};
    T* bstage_out[2] = {};
    double* bnorms_h = nullptr;  // pinned: per solve max_iters+1 norms + 2 state ints (as doubles)
    int bnorms_cap = 0;

    int batch_init(int per_solve, int nrhs) {
        if (!bs_h2d) {
            CK(cudaStreamCreateWithFlags(&bs_h2d, cudaStreamNonBlocking));
            CK(cudaStreamCreateWithFlags(&bs_d2h, cudaStreamNonBlocking));
            for (int i = 0; i < 2; ++i) {
                CK(cudaEventCreateWithFlags(&ev_in[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_pad[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_unpad[i], cudaEventDisableTiming));
                CK(cudaEventCreateWithFlags(&ev_out[i], cudaEventDisableTiming));
                const size_t cnt = (size_t)count_of(cfg.dim, cfg.N);
                if (int rc = dalloc(&bstage_in[i], cnt)) return rc;
                if (int rc = dalloc(&bstage_out[i], cnt)) return rc;
            }
            CK(cudaEventCreateWithFlags(&ev_go, cudaEventDisableTiming));
        }
        if (per_solve * nrhs > bnorms_cap) {
            if (bnorms_h) cudaFreeHost(bnorms_h);
            bnorms_h = nullptr;
            CK(cudaMallocHost(&bnorms_h, sizeof(double) * per_solve * nrhs));
            bnorms_cap = per_solve * nrhs;
        }
        return 0;
    }

    int solve_batch(int nrhs, const void* const* bh, void* const* uh, double tol, int max_iters, double* norms,
                    int* iters, int* conv, cudaStream_t s) override {
        if (int rc = grow_norms(max_iters + 1)) return rc;
        hist_len = 0;
        if (nrhs <= 0) return 0;
        if (!use_graph) return fail(SPAIMG_ENOTSUP, "solve_batch needs the graph path");
        if (!exec_solve)
            if (int rc = build_solve_graph()) return rc;
        const int per = max_iters + 1 + 2;
        if (int rc = batch_init(per, nrhs)) return rc;
        const size_t bytes = (size_t)count_of(cfg.dim, cfg.N) * sizeof(T);
        Level<T>& L0 = lv[0];
        ctl_h->tol = tol;
        ctl_h->max_iters = max_iters;
        CK(cudaMemcpyAsync(ctl_d, ctl_h, sizeof(SolveCtl), cudaMemcpyHostToDevice, s));
        CK(cudaEventRecord(ev_go, s));
        CK(cudaStreamWaitEvent(bs_h2d, ev_go, 0));
        CK(cudaStreamWaitEvent(bs_d2h, ev_go, 0));
        // cudaMemcpyDefault: the right-hand sides and outputs may be host or device arrays
        CK(cudaMemcpyAsync(bstage_in[0], bh[0], bytes, cudaMemcpyDefault, bs_h2d));
        CK(cudaEventRecord(ev_in[0], bs_h2d));
        for (int i = 0; i < nrhs; ++i) {
            const int c = i & 1, o = c ^ 1;
            if (i + 1 < nrhs) {  // prefetch the next right-hand side once its stage is free
                if (i >= 1) CK(cudaStreamWaitEvent(bs_h2d, ev_pad[o], 0));
                CK(cudaMemcpyAsync(bstage_in[o], bh[i + 1], bytes, cudaMemcpyDefault, bs_h2d));
                CK(cudaEventRecord(ev_in[o], bs_h2d));
            }
            CK(cudaStreamWaitEvent(s, ev_in[c], 0));
            CK(launch_pad<T>(L0.L, bstage_in[c], L0.b, s));
            CK(cudaEventRecord(ev_pad[c], s));
            CK(cudaMemsetAsync(L0.x[0], 0, (size_t)L0.L.alloc * sizeof(T), s));
            CK(cudaGraphLaunch(exec_solve, s));
            CK(cudaMemcpyAsync(bnorms_h + (size_t)i * per, norms_d, sizeof(double) * (max_iters + 1),
                               cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(bnorms_h + (size_t)i * per + max_iters + 1, state_d, 2 * sizeof(int),
                               cudaMemcpyDeviceToHost, s));
            if (i >= 2) CK(cudaStreamWaitEvent(s, ev_out[c], 0));  // solution i-2 left this stage
            CK(launch_unpad<T>(L0.L, L0.x[0], bstage_out[c], s));
            CK(cudaEventRecord(ev_unpad[c], s));
            CK(cudaStreamWaitEvent(bs_d2h, ev_unpad[c], 0));
            CK(cudaMemcpyAsync(uh[i], bstage_out[c], bytes, cudaMemcpyDefault, bs_d2h));
            CK(cudaEventRecord(ev_out[c], bs_d2h));
        }
        CK(cudaStreamWaitEvent(s, ev_out[(nrhs - 1) & 1], 0));
        CK(cudaStreamSynchronize(s));
        for (int i = 0; i < nrhs; ++i) {
            const double* h = bnorms_h + (size_t)i * per;
            int st[2];
            std::memcpy(st, h + max_iters + 1, sizeof(st));
            iters[i] = st[0];
            conv[i] = st[1];
            for (int k = 0; k <= st[0]; ++k) norms[(size_t)i * (max_iters + 1) + k] = h[k];
        }
        return 0;
    }

    int op_launch(int which, cudaStream_t s) {
        Level<T>& L = lv[0];
        if (nsmooth() < 1) return fail(SPAIMG_EINVAL, "no smoothing level");
        int launches = 0;
        switch (which) {
            case 0: return do_sweep<T>(L, 0, false, M, shape, fused, omega, s, nullptr);
            case 1: CK(launch_residual_restrict<T>(L.L, lv[1].L, L.x[0], L.b, lv[1].b, L.sA, s)); return 0;
            case 2: CK(launch_prolong_correct<T>(L.L, lv[1].L, L.x[1], L.x[1], lv[1].x[0], s)); return 0;
            case 3: {
                // keep the history cursor in range while timing repeated norms
                CK(cudaMemsetAsync(slot_d, 0, sizeof(int), s));
                return norm_launch(L.x[0], s, &launches);
            }
            case 4: {  // fused sweep + norm (part A)
                CK(cudaMemsetAsync(slot_d, 0, sizeof(int), s));
                return part_a(s, &launches);
            }
            case 5:  // two sweeps in one march (2D marching levels)
                CK(launch_sweep2<T>(L.L, L.x[0], L.b, L.x[1], M, shape, L.sA, L.sM, omega, false, s));
                return 0;
            case 6:  // K3 + K1: sweep(x + P e) in one march (levels where sweep_pc_supported)
                if (!fused || !sweep_pc_supported(L.L, shape)) return fail(SPAIMG_ENOTSUP, "no K3 + K1 march on this level");
                CK(launch_sweep_pc<T>(L.L, lv[1].L, L.x[0], lv[1].x[0], L.b, L.x[1], M, shape, L.sA, L.sM, omega, s));
                return 0;
            default: return fail(SPAIMG_EINVAL, "unknown op");
        }
    }

    // `reps` back-to-back launches of one kernel, replayed from a cached CUDA graph so the
    // per-launch time excludes host launch gaps (used for per-operator timing)
    int op(int which, int reps, cudaStream_t s) override {
        if (reps <= 1) return reps == 1 ? op_launch(which, s) : 0;
        const long long key = (long long)which * 1000003 + reps;
        for (auto& kv : op_graphs)
            if (kv.first == key) {
                CK(cudaGraphLaunch(kv.second, s));
                return 0;
            }
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        int rc = capture_into(g, [&](cudaStream_t cs) -> int {
            for (int k = 0; k < reps; ++k)
                if (int r = op_launch(which, cs)) return r;
            return 0;
        });
        cudaGraphExec_t ex = nullptr;
        if (!rc) {
            cudaError_t e = cudaGraphInstantiate(&ex, g, 0);
            if (e != cudaSuccess) rc = fail((int)e, "op graph instantiate failed");
        }
        cudaGraphDestroy(g);
        if (rc) return rc;
        op_graphs.push_back({key, ex});
        CK(cudaGraphLaunch(ex, s));
        return 0;
    }

    void stats(spaimg_solver_stats* st) const override {
        st->levels = nsmooth();
        st->kernels_per_cycle = kernels_per_cycle;
        st->kernels_stop_test = kernels_a;
        st->unknowns = count_of(cfg.dim, cfg.N);
        st->graph = use_graph ? 1 : 0;
        st->fused_sweep = fused ? 1 : 0;
        // per visit of level l: n_l s (3(nu1+nu2) + 4 + 2^(1-d)); + 2 s n_0 (norm)
        const double sz = sizeof(T);
        double bytes = 2.0 * sz * (double)count_of(cfg.dim, cfg.N);
        double visits = 1.0;
        for (int l = 0; l < nsmooth(); ++l) {
            const double nl = (double)count_of(cfg.dim, lv[l].L.N);
            bytes += visits * nl * sz * (3.0 * (cfg.nu1 + cfg.nu2) + 4.0 + std::pow(2.0, 1 - cfg.dim));
            visits *= cfg.gamma;
        }
        st->bytes_per_cycle = bytes;
    }
};

static int check_cfg(const spaimg_mg_config* c) {
    if (!c) return fail(SPAIMG_EINVAL, "config is NULL");
    if (int rc = check_dims(c->dtype, c->dim, c->N)) return rc;
    if (int rc = check_stencil(&c->M, c->dim)) return rc;
    if (c->gamma != 1 && c->gamma != 2) return fail(SPAIMG_EINVAL, "gamma must be 1 (V) or 2 (W)");
    if (c->nu1 < 0 || c->nu2 < 0 || c->nu1 + c->nu2 < 1) return fail(SPAIMG_EINVAL, "need nu1, nu2 >= 0 with nu1 + nu2 >= 1");
    if (c->coarsest_N < 2) return fail(SPAIMG_EINVAL, "coarsest_N must be at least 2");
    if (!c->coarse_lu || !c->coarse_piv || c->coarse_n < 1) return fail(SPAIMG_EINVAL, "missing coarse factorisation");
    return 0;
}

extern "C" int spaimg_solver_create(const spaimg_mg_config* cfg, spaimg_solver** out) {
    if (int rc = check_cfg(cfg)) return rc;
    if (!out) return fail(SPAIMG_EINVAL, "out is NULL");
    std::unique_ptr<spaimg_solver> s;
    int rc;
    if (cfg->dtype == SPAIMG_F64) {
        auto p = std::make_unique<Solver<double>>();
        rc = p->init(*cfg);
        s = std::move(p);
    } else {
        auto p = std::make_unique<Solver<float>>();
        rc = p->init(*cfg);
        s = std::move(p);
    }
    if (rc) return rc;
    *out = s.release();
    return 0;
}

extern "C" int spaimg_solver_destroy(spaimg_solver* s) {
    delete s;
    return 0;
}

extern "C" int spaimg_solver_stats_get(const spaimg_solver* s, spaimg_solver_stats* st) {
    if (!s || !st) return fail(SPAIMG_EINVAL, "NULL argument");
    s->stats(st);
    return 0;
}

extern "C" int spaimg_solver_load(spaimg_solver* s, const void* b, const void* u0, void* stream) {
    if (!s) return fail(SPAIMG_EINVAL, "NULL solver");
    return s->load(b, u0, (cudaStream_t)stream);
}

extern "C" int spaimg_solver_cycles(spaimg_solver* s, int ncycles, void* stream) {
    if (!s) return fail(SPAIMG_EINVAL, "NULL solver");
    return s->cycles(ncycles, (cudaStream_t)stream);
}

extern "C" int spaimg_solver_run(spaimg_solver* s, double tol, int max_iters, double* norms, int* iterations,
                                 int* converged, void* stream) {
    if (!s || !norms || !iterations || !converged) return fail(SPAIMG_EINVAL, "NULL argument");
    if (max_iters < 0) return fail(SPAIMG_EINVAL, "max_iters must be non-negative");
    return s->run(tol, max_iters, norms, iterations, converged, (cudaStream_t)stream);
}

extern "C" int spaimg_solver_solve_batch(spaimg_solver* s, int nrhs, const void* const* b, void* const* u_out,
                                         double tol, int max_iters, double* norms, int* iterations, int* converged,
                                         void* stream) {
    if (!s || (nrhs > 0 && (!b || !u_out || !norms || !iterations || !converged)))
        return fail(SPAIMG_EINVAL, "NULL argument");
    if (nrhs < 0 || max_iters < 0) return fail(SPAIMG_EINVAL, "nrhs and max_iters must be non-negative");
    for (int i = 0; i < nrhs; ++i)
        if (!b[i] || !u_out[i]) return fail(SPAIMG_EINVAL, "NULL right-hand side or output");
    return s->solve_batch(nrhs, b, u_out, tol, max_iters, norms, iterations, converged, (cudaStream_t)stream);
}

extern "C" int spaimg_fill_uniform(int dtype, long long count, unsigned long long state_hi,
                                   unsigned long long state_lo, unsigned long long inc_hi, unsigned long long inc_lo,
                                   double low, double high, void* out, void* stream) {
    if (dtype != SPAIMG_F64 && dtype != SPAIMG_F32) return fail(SPAIMG_EINVAL, "dtype must be SPAIMG_F64 or SPAIMG_F32");
    if (count < 0 || (count > 0 && !out)) return fail(SPAIMG_EINVAL, "bad output");
    if (!is_device_ptr(out)) return fail(SPAIMG_EINVAL, "spaimg_fill_uniform writes device memory");
    const unsigned long long st[4] = {state_hi, state_lo, inc_hi, inc_lo};
    cudaStream_t s = (cudaStream_t)stream;
    CK(dtype == SPAIMG_F64 ? launch_fill_uniform<double>(static_cast<double*>(out), count, st, low, high, s)
                           : launch_fill_uniform<float>(static_cast<float*>(out), count, st, low, high, s));
    return 0;
}

extern "C" int spaimg_solver_store(spaimg_solver* s, void* u_out, void* stream) {
    if (!s || !u_out) return fail(SPAIMG_EINVAL, "NULL argument");
    return s->store(u_out, (cudaStream_t)stream);
}

extern "C" int spaimg_solver_op(spaimg_solver* s, int op, int reps, void* stream) {
    if (!s) return fail(SPAIMG_EINVAL, "NULL solver");
    return s->op(op, reps, (cudaStream_t)stream);
}

extern "C" int spaimg_cycle(const spaimg_mg_config* cfg, const void* u, const void* b, void* out, void* stream) {
    spaimg_solver* s = nullptr;
    if (int rc = spaimg_solver_create(cfg, &s)) return rc;
    std::unique_ptr<spaimg_solver> own(s);
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = s->load(b, u, st)) return rc;
    if (int rc = s->cycles(1, st)) return rc;
    return s->store(out, st);
}

extern "C" int spaimg_solve(const spaimg_mg_config* cfg, const void* b, const void* u0, void* u_out, double tol,
                            int max_iters, double* norms, int* iterations, int* converged, void* stream) {
    spaimg_solver* s = nullptr;
    if (int rc = spaimg_solver_create(cfg, &s)) return rc;
    std::unique_ptr<spaimg_solver> own(s);
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = s->load(b, u0, st)) return rc;
    if (int rc = s->run(tol, max_iters, norms, iterations, converged, st)) return rc;
    return s->store(u_out, st);
}
