/* C restatement of the spaimg V-cycle hot path — TEST INFRASTRUCTURE ONLY.
 *
 * Used by tests/ as a checker and by bench.py as the CPU baseline; never linked into
 * the product library.  Restates reference pkg/src/spaimg/stencils.py:136-153 and
 * multigrid.py:86-227 following SURVEY.md Appendix A.  Build: `make -C oracle`
 * (gcc -O2 -fopenmp -ffp-contract=off; contraction would break bitwise parity).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define REAL double
#define SFX _f64
#define FMA fma
#include "spaimg_oracle_impl.h"
#undef REAL
#undef SFX
#undef FMA

#define REAL float
#define SFX _f32
#define FMA fmaf
#include "spaimg_oracle_impl.h"
#undef REAL
#undef SFX
#undef FMA

#ifdef _OPENMP
#include <omp.h>
int oracle_max_threads(void) { return omp_get_max_threads(); }
void oracle_set_threads(int n) { omp_set_num_threads(n); }
#else
int oracle_max_threads(void) { return 1; }
void oracle_set_threads(int n) { (void)n; }
#endif
