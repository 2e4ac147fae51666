/* spaimg_cuda.h — C ABI of the B200 (sm_100a) geometric-multigrid hot path.
 *
 * Drop-in boundary for the reference package `spaimg` (arXiv 2206.05543).  The reference has
 * no FFI of its own: its boundary is the Python function API of spaimg.multigrid, re-exported
 * at pkg/src/spaimg/__init__.py:21, plus Stencil.apply (stencils.py:136).  Each entry point
 * below replaces exactly one of those functions; the Python mirror in
 * paper_2206_05543_b200/multigrid.py binds them with ctypes (INTEGRATION.md shows the stub a
 * maintainer would add to the reference itself).
 *
 * Conventions
 *   - Arrays are the reference's Grid.values layout: (N-1)^dim values, C order (grids.py:10-56).
 *     Pointers may be device pointers (cudaMalloc / torch CUDA tensors) or host pointers
 *     (pageable or pinned); the kind is detected with cudaPointerGetAttributes.  Host outputs
 *     are complete when the call returns; device outputs are stream-ordered on `stream`.
 *   - dtype: SPAIMG_F64 (the reference's only precision, grids.py:24) or SPAIMG_F32 (build
 *     contract of SURVEY.md Appendix A.8).
 *   - stream: a cudaStream_t (e.g. torch.cuda.current_stream().cuda_stream), NULL = legacy.
 *   - Return value 0 on success; < 0 for an argument error (SPAIMG_E*), > 0 a cudaError_t.
 *     spaimg_last_error() returns a thread-local message for the last failure.  The Python
 *     mirror validates first and raises the reference's ValueError/TypeError messages, so a
 *     non-zero return from here is a bug or a device fault.
 *   - Arithmetic: every output is bitwise identical to the reference's numpy expression
 *     trees (no FMA contraction except where the reference's BLAS uses it, Appendix A.6).
 */
#ifndef SPAIMG_CUDA_H
#define SPAIMG_CUDA_H

#ifdef __cplusplus
extern "C" {
#endif

#define SPAIMG_ABI_VERSION 1

#if defined(__GNUC__)
#define SPAIMG_API __attribute__((visibility("default")))
#else
#define SPAIMG_API
#endif

#define SPAIMG_F64 0
#define SPAIMG_F32 1

#define SPAIMG_EINVAL (-1)   /* bad argument (shape, N, dim, config) */
#define SPAIMG_ENOTSUP (-2)  /* an unsupported request (dtype, engine limits) */

#define SPAIMG_MAX_TERMS 27

/* One stencil: reference Stencil(dim, entries, h_exponent), stencils.py:73-92.  offsets/coef
 * list the entries in dict insertion order with coef[k] = float(c) (stencils.py:149-151). */
typedef struct spaimg_stencil {
    int dim;
    int nterms;
    int h_exponent;
    int offsets[SPAIMG_MAX_TERMS][3];
    double coef[SPAIMG_MAX_TERMS];
} spaimg_stencil;

/* A resolved MgConfig (multigrid.py:30-68) for one problem size. */
typedef struct spaimg_mg_config {
    int dtype;
    int dim;
    int N;              /* finest mesh count (Grid.N) */
    spaimg_stencil M;   /* MgConfig.resolve_smoother()[0] */
    double omega;       /* MgConfig.resolve_smoother()[1] */
    int gamma;          /* 1 = "V", 2 = "W" (multigrid.py:173) */
    int nu1, nu2;
    int coarsest_N;
    /* lu_factor(laplacian(dim).to_matrix(coarse_N).toarray()) (multigrid.py:147-149), where
     * coarse_N is the first mesh count <= coarsest_N reached by halving N. */
    int coarse_N;
    int coarse_n;              /* (coarse_N-1)^dim */
    const double *coarse_lu;   /* host, row-major coarse_n x coarse_n */
    const int *coarse_piv;     /* host, 0-based row interchanges */
} spaimg_mg_config;

typedef struct spaimg_solver spaimg_solver;

typedef struct spaimg_solver_stats {
    int levels;              /* smoothing levels (excluding the coarse solve level) */
    int kernels_per_cycle;   /* kernel launches per cycle of the device-side solve loop (incl. norm + stop test) */
    double bytes_per_cycle;  /* SURVEY.md §8d minimal algorithmic bytes of one cycle + norm */
    long long unknowns;      /* (N-1)^dim on the finest level */
    int graph;               /* 1 if cycles replay a CUDA graph */
    int fused_sweep;         /* 1 if the fused K1 sweep is used for this smoother */
    int kernels_stop_test;   /* launches of the per-cycle norm + stop-test part (also run once
                                more after the last cycle): a solve of K cycles launches
                                1 + K*kernels_per_cycle + kernels_stop_test kernels */
} spaimg_solver_stats;

SPAIMG_API const char *spaimg_last_error(void);
SPAIMG_API int spaimg_abi_version(void);
/* select the CUDA device for subsequent calls from this thread (the library links its own
 * CUDA runtime, so the caller's device choice, e.g. torch.cuda.current_device(), is forwarded) */
SPAIMG_API int spaimg_set_device(int device);

/* Stencil.apply (stencils.py:136-153): out = h^e * sum_k c_k x[i+o_k], zero extension. */
SPAIMG_API int spaimg_apply(int dtype, int N, const spaimg_stencil *S, const void *x, void *out, void *stream);

/* smooth(u, b, M, omega, steps) (multigrid.py:86-101). */
SPAIMG_API int spaimg_smooth(int dtype, int dim, int N, const void *u, const void *b, const spaimg_stencil *M,
                  double omega, int steps, void *out, void *stream);

/* restrict(fine) (multigrid.py:110-119): N even, N/2 >= 2; coarse has (N/2-1)^dim values. */
SPAIMG_API int spaimg_restrict(int dtype, int dim, int N, const void *fine, void *coarse, void *stream);

/* prolong(coarse, fine_N) (multigrid.py:133-144): fine_N == 2*coarse_N. */
SPAIMG_API int spaimg_prolong(int dtype, int dim, int coarse_N, const void *coarse, void *fine, void *stream);

/* Fused building blocks of cycle(): restrict(b - A u) (multigrid.py:176-177) and
 * u + prolong(e, N) (multigrid.py:184). */
SPAIMG_API int spaimg_residual_restrict(int dtype, int dim, int N, const void *u, const void *b, void *coarse,
                             void *stream);
SPAIMG_API int spaimg_prolong_correct(int dtype, int dim, int N, const void *u, const void *e, void *out, void *stream);

/* ||b - A u||_2 (multigrid.py:207, :214); *out is written before return. */
SPAIMG_API int spaimg_residual_norm(int dtype, int dim, int N, const void *u, const void *b, double *out, void *stream);

/* cycle(u, b, cfg) (multigrid.py:157-185). */
SPAIMG_API int spaimg_cycle(const spaimg_mg_config *cfg, const void *u, const void *b, void *out, void *stream);

/* solve(b, cfg) loop (multigrid.py:203-219) from the start u0 (NULL = zero).  norms receives
 * ||r_0|| .. ||r_K|| (room for max_iters+1 doubles, host); u_out receives the final iterate. */
SPAIMG_API int spaimg_solve(const spaimg_mg_config *cfg, const void *b, const void *u0, void *u_out, double tol,
                 int max_iters, double *norms, int *iterations, int *converged, void *stream);

/* Reusable solver: owns the padded level hierarchy and the captured cycle graph. */
SPAIMG_API int spaimg_solver_create(const spaimg_mg_config *cfg, spaimg_solver **out);
SPAIMG_API int spaimg_solver_destroy(spaimg_solver *s);
SPAIMG_API int spaimg_solver_stats_get(const spaimg_solver *s, spaimg_solver_stats *st);
/* load b (NULL = keep the loaded one) and the start u0 (NULL = zero) into the finest level */
SPAIMG_API int spaimg_solver_load(spaimg_solver *s, const void *b, const void *u0, void *stream);
/* run `ncycles` cycles without reading anything back (each appends its norm on device) */
SPAIMG_API int spaimg_solver_cycles(spaimg_solver *s, int ncycles, void *stream);
/* full solve loop on the loaded problem */
SPAIMG_API int spaimg_solver_run(spaimg_solver *s, double tol, int max_iters, double *norms, int *iterations,
                      int *converged, void *stream);
/* numpy Generator(PCG64).uniform(low, high, count) in C order into device memory, bitwise: the
 * reference solve()'s random start default_rng(rng_seed).uniform(0, 1, shape) (multigrid.py:204-205)
 * without a host draw or upload.  (state, inc) = the seeded generator's 128-bit PCG64 state
 * (numpy: default_rng(seed).bit_generator.state), split into 64-bit halves. */
SPAIMG_API int spaimg_fill_uniform(int dtype, long long count, unsigned long long state_hi,
                                   unsigned long long state_lo, unsigned long long inc_hi, unsigned long long inc_lo,
                                   double low, double high, void *out, void *stream);

/* copy the current finest iterate out (dense layout) */
SPAIMG_API int spaimg_solver_store(spaimg_solver *s, void *u_out, void *stream);
/* nrhs independent zero-start solves of the solver's problem (solve() loop of multigrid.py:206-219
 * per right-hand side), pipelined: b[i+1] is copied in and u_out[i-1] copied out on their own
 * streams while solve i runs.  b[i] / u_out[i]: dense (N-1)^dim arrays, host (pinned for the
 * overlap) or device.  norms: nrhs x (max_iters+1) row-major (row i holds ||r_0|| .. ||r_k||);
 * iterations / converged: nrhs each.  Returns when every output has landed. */
SPAIMG_API int spaimg_solver_solve_batch(spaimg_solver *s, int nrhs, const void *const *b, void *const *u_out,
                                         double tol, int max_iters, double *norms, int *iterations, int *converged,
                                         void *stream);

/* Isolated kernel launches on the solver's finest-level buffers, for per-operator timing
 * (BASELINE.json config 5): op 0 = fused sweep (K1), 1 = residual+restriction (K2),
 * 2 = prolongation+correction (K3), 3 = residual norm (K4), 4 = norm + first pre-sweep (part A of
 * the solve loop), 5 = two sweeps in one march (2D marching levels, C1 / STAR5 shapes),
 * 6 = prolongation+correction fused into the sweep (K3+K1; SPAIMG_ENOTSUP where the level does
 * not use it).  `reps` back-to-back launches, replayed from a cached graph. */
SPAIMG_API int spaimg_solver_op(spaimg_solver *s, int op, int reps, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* SPAIMG_CUDA_H */
