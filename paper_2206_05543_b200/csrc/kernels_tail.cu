// K5+: the shared-memory coarse-grid engine.  All levels from a size threshold down (2D n <= 63,
// 3D n <= 15) live in ONE CTA's shared memory, and the CTA runs the whole V/W recursion below
// its entry level (reference multigrid.py:157-185) without leaving the SM:
//   1. load the host-recorded op list and the coarse LU data into shared memory, copy the entry
//      level's b and start iterate (with their zero frames) from global memory, zero the rest;
//   2. interpret the ops, each point-parallel over its level; consecutive ops are separated by a
//      barrier over only the warps involved (__syncwarp for one warp, a named barrier per
//      distinct warp count, __syncthreads for all) -- the small levels of a W-cycle run on one
//      or two warps and do not pay for a 16-warp barrier;
//   3. store the entry level's iterate back to global memory (in place).
// Point mapping: a level's interior is embedded in a W^dim box (W = 1 << logw >= n); thread t
// owns one position of the box's (dim-1)-dimensional cross-section and a strip of K consecutive
// points along axis 0 (K = W^dim / 512 for the big levels, else 1), so a stencil's loads along
// axis 0 are shared between the strip's points (register tile) instead of re-read from shared
// memory (shared-memory bandwidth, 128 B/clk/SM, bounds the big levels).
// Every per-point expression is the Appendix-A tree of the multi-kernel path
// (spaimg_common.cuh), so the engine is bitwise identical to it; only the memory changes.  The
// relaxation updates x in place: x' at a point reads x only at that point (multigrid.py:100).
#include "tail_ops.cuh"

namespace spaimg {

// ------------------------------------------------------------------------------------------
// the engine
// ------------------------------------------------------------------------------------------
__device__ __forceinline__ void tail_barrier(int bid, int bw) {
    if (bid == 0) {
        __syncthreads();
    } else if (bid == kTailSyncWarp) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(bid), "r"(bw * 32) : "memory");
    }
}

template <class T, int S, int D, int LOGW>
__device__ __forceinline__ void run_point_op(int type, const TailArgs<T>& a, int lev, T* arr, int i) {
    const TailLv<T>& f = a.lv[lev];
    if (a.prof && threadIdx.x == 0) a.prof[kTailMaxOps + i] = clock64();
    switch (type) {
        case TAIL_RES: op_res<T, D, LOGW>(f, arr); break;
        case TAIL_RELAX: op_relax<T, S, D, LOGW, false>(f, arr, a.M, a.omega); break;
        case TAIL_RELAX0: op_relax<T, S, D, LOGW, true>(f, arr, a.M, a.omega); break;
        case TAIL_ZERO: op_zero<T, D, LOGW>(f, arr); break;
        case TAIL_FW: op_fw<T, D, LOGW>(f, a.lv[lev + 1], arr); break;
        case TAIL_PROLONG: op_prolong<T, D, LOGW>(f, a.lv[lev + 1], arr); break;
        default: break;
    }
}

template <class T, int S, int D>
__global__ void __launch_bounds__(NT, 1) k_tail(const __grid_constant__ TailArgs<T> a) {
    extern __shared__ __align__(16) unsigned char smem[];
    T* arr = reinterpret_cast<T*>(smem);
    const int nlu = a.nlu;
    // nlu > kTailMaxLU: the factors and the work vector follow the level arrays
    T* cf = arr + a.arr_elems;
    int* ci = reinterpret_cast<int*>(cf + (nlu > kTailMaxLU ? nlu * nlu + 2 * nlu : 0));
    T* ywork = reinterpret_cast<T*>(ci + (nlu > kTailMaxLU ? 2 * nlu + 2 : 0));
    const int t = threadIdx.x;

    // 1. the entry level (frames included), zeroed scratch, large coarse factors
    {
        const TailLv<T>& e = a.lv[0];
        tail_load_entry<T, D>(a, arr, e.x, e.b, e.s0, e.s1);
        for (int i = a.zero_from + t; i < a.arr_elems; i += NT) arr[i] = T(0);
        if constexpr (kDebugChecks) {
            // NaN interiors (zero frames) for every array the engine writes before reading
            __syncthreads();
            for (int l = 0; l < a.nlv; ++l) {
                const TailLv<T>& g = a.lv[l];
                const int F = a.frame;
                tail_poison<T, D>(arr, g.n, F, g.s0, g.s1, l == 0 ? -1 : g.x);
                tail_poison<T, D>(arr, g.n, F, g.s0, g.s1, l == 0 ? -1 : g.b);
                if (g.r >= 0) tail_poison<T, D>(arr, g.n, F, g.s0, g.s1, g.r);
            }
        }
        if (nlu > kTailMaxLU) {
            for (int i = t; i < nlu * nlu + 2 * nlu; i += NT) cf[i] = a.coarse_g[i];
            for (int i = t; i < 2 * nlu; i += NT) ci[i] = a.coarse_idx_g[i];
        }
    }
    __syncthreads();

    // 2. the op list
    const int warp = t >> 5;
    for (int i = 0; i < a.nops; ++i) {
        const unsigned w = a.ops[i];
        const int type = w & 7, lev = (w >> 3) & 7, nw = (w >> 6) & 31, bw = (w >> 11) & 31, bid = (w >> 16) & 31;
        if (warp >= bw) continue;
        if (i > 0) tail_barrier(bid, bw);
        SPAIMG_JITTER();
        if (a.prof && t == 0) a.prof[i] = clock64();
        if (warp >= nw) continue;
        if (type == TAIL_COARSE) {
            constexpr int NLU = D == 2 ? 9 : 27;  // coarsest_N = 4
            const TailLv<T>& c = a.lv[lev];
            if (nlu == 1)
                coarse_thread<T, 1>(a, c, arr);
            else if (nlu == NLU)
                coarse_thread<T, NLU>(a, c, arr);
            else if (nlu <= kTailMaxLU)
                coarse_warp<T>(a, c, arr);
            else
                coarse_block<T>(c, arr, cf, ci, nlu, ywork);
            continue;
        }
        const int logw = a.lv[lev].logw;
        if (D == 2) {
            switch (logw) {
                case 2: run_point_op<T, S, D, 2>(type, a, lev, arr, i); break;
                case 3: run_point_op<T, S, D, 3>(type, a, lev, arr, i); break;
                case 4: run_point_op<T, S, D, 4>(type, a, lev, arr, i); break;
                case 5: run_point_op<T, S, D, 5>(type, a, lev, arr, i); break;
                case 6: run_point_op<T, S, D, 6>(type, a, lev, arr, i); break;
                default: break;
            }
        } else {
            switch (logw) {
                case 2: run_point_op<T, S, D, 2>(type, a, lev, arr, i); break;
                case 3: run_point_op<T, S, D, 3>(type, a, lev, arr, i); break;
                case 4: run_point_op<T, S, D, 4>(type, a, lev, arr, i); break;
                default: break;
            }
        }
        if (a.prof && t == 0) a.prof[2 * kTailMaxOps + i] = clock64();
    }
    __syncthreads();
    if (a.prof && t == 0) a.prof[a.nops] = clock64();

    // 3. the entry level's iterate back to global memory (interior only)
    tail_store_entry<T, D>(a, arr, a.lv[0].x, a.lv[0].s0, a.lv[0].s1);
}

template <class T, int S, int D>
static cudaError_t launch_tail_s(const TailArgs<T>& a, cudaStream_t s) {
    if (a.smem > 48 * 1024) {  // per device, so set on every launch (host-side, cheap)
        cudaError_t e = cudaFuncSetAttribute(k_tail<T, S, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)a.smem);
        if (e != cudaSuccess) return e;
    }
    return launch_k(k_tail<T, S, D>, dim3(1), dim3(NT), a.smem, s, a);
}

template <class T>
cudaError_t launch_tail(const TailArgs<T>& a, cudaStream_t s) {
    if (a.fast_le > 0) return a.gL.dim == 2 ? launch_tail_fast2d<T>(a, s) : launch_tail_fast3d<T>(a, s);
    if (a.gL.dim == 2) {
        switch (a.shape) {
            case SHAPE_C1: return launch_tail_s<T, SHAPE_C1, 2>(a, s);
            case SHAPE_STAR5: return launch_tail_s<T, SHAPE_STAR5, 2>(a, s);
            case SHAPE_BOX9: return launch_tail_s<T, SHAPE_BOX9, 2>(a, s);
            default: return launch_tail_s<T, SHAPE_GENERIC, 2>(a, s);
        }
    }
    switch (a.shape) {
        case SHAPE_C1: return launch_tail_s<T, SHAPE_C1, 3>(a, s);
        case SHAPE_STAR7: return launch_tail_s<T, SHAPE_STAR7, 3>(a, s);
        default: return launch_tail_s<T, SHAPE_GENERIC, 3>(a, s);
    }
}

template cudaError_t launch_tail<double>(const TailArgs<double>&, cudaStream_t);
template cudaError_t launch_tail<float>(const TailArgs<float>&, cudaStream_t);

}  // namespace spaimg
