// Launch-latency probe (not part of the library): per-node cost of dependent kernel chains in a
// CUDA graph (plain, with PDL, inside a conditional WHILE body) and of a software grid barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/latency_probe tools/latency_probe.cu && /tmp/latency_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p) atomicAdd(p, 1);
}
__global__ void k_empty_pdl(int* p) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0 && blockIdx.x == 0 && p) atomicAdd(p, 1);
    asm volatile("griddepcontrol.launch_dependents;");
}

struct Big {
    double c[96];
};
__global__ void k_big(int* p, Big b) {
    if (threadIdx.x == 0 && blockIdx.x == 0 && p && b.c[5] > 1e300) atomicAdd(p, 1);
}

__device__ __forceinline__ void grid_sync(unsigned* bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned* gen = bar + 1;
        const unsigned g = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g) {
            }
        }
        __threadfence();
    }
    __syncthreads();
}
__global__ void k_barriers(unsigned* bar, int n) {
    for (int i = 0; i < n; ++i) grid_sync(bar);
}

__global__ void k_set(int* c, int v) { *c = v; }
__global__ void k_dec(int* c, cudaGraphConditionalHandle h) {
    int v = --*c;
    cudaGraphSetConditional(h, v > 0 ? 1u : 0u);
}

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e));               \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

static float time_graph(cudaGraphExec_t ge, cudaStream_t s, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEventRecord(a, s);
    for (int i = 0; i < reps; ++i) cudaGraphLaunch(ge, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    int* d;
    CK(cudaMalloc(&d, 64));
    const int K = 100;
    for (int blocks : {1, 148, 592}) {
        for (int pdl = 0; pdl < 2; ++pdl) {
            cudaGraph_t g;
            CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
            for (int i = 0; i < K; ++i) {
                cudaLaunchConfig_t cfg{};
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(256);
                cfg.stream = s;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = 1;
                cfg.attrs = at;
                cfg.numAttrs = pdl;
                if (pdl)
                    CK(cudaLaunchKernelEx(&cfg, k_empty_pdl, (int*)nullptr));
                else
                    CK(cudaLaunchKernelEx(&cfg, k_empty, (int*)nullptr));
            }
            CK(cudaStreamEndCapture(s, &g));
            cudaGraphExec_t ge;
            CK(cudaGraphInstantiate(&ge, g, 0));
            float ms = time_graph(ge, s, 20);
            printf("chain of %d empty kernels, %d CTAs, pdl=%d: %.3f us per kernel\n", K, blocks, pdl, ms * 1e3 / K);
        }
    }
    // inside a conditional WHILE body (10 iterations x 10 kernels)
    {
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams p{};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        // set counter node
        cudaGraphNode_t nset, ncond;
        cudaKernelNodeParams kp{};
        int v = 10;
        void* args_set[] = {&d, &v};
        kp.func = (void*)k_set;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args_set;
        CK(cudaGraphAddKernelNode(&nset, g, nullptr, 0, &kp));
        CK(cudaGraphAddNode(&ncond, g, &nset, 1, &p));
        cudaGraph_t body = p.conditional.phGraph_out[0];
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < 10; ++i) k_empty<<<148, 256, 0, cs>>>(nullptr);
        k_dec<<<1, 1, 0, cs>>>(d, h);
        CK(cudaStreamEndCapture(cs, &body));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        float ms = time_graph(ge, s, 20);
        printf("WHILE body (10 iters x 11 kernels, 148 CTAs): %.3f us per kernel\n", ms * 1e3 / 110);
    }
    // 768-byte kernel parameters: flat chain and inside a WHILE body
    {
        Big bg{};
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < K; ++i) k_big<<<148, 256, 0, s>>>(nullptr, bg);
        CK(cudaStreamEndCapture(s, &g));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        printf("chain of %d 768-B-param kernels, 148 CTAs: %.3f us per kernel\n", K, time_graph(ge, s, 20) * 1e3 / K);
    }
    {
        Big bg{};
        cudaGraph_t g;
        CK(cudaGraphCreate(&g, 0));
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
        cudaGraphNodeParams p{};
        p.type = cudaGraphNodeTypeConditional;
        p.conditional.handle = h;
        p.conditional.type = cudaGraphCondTypeWhile;
        p.conditional.size = 1;
        cudaGraphNode_t nset, ncond;
        cudaKernelNodeParams kp{};
        int v = 10;
        void* args_set[] = {&d, &v};
        kp.func = (void*)k_set;
        kp.gridDim = dim3(1);
        kp.blockDim = dim3(1);
        kp.kernelParams = args_set;
        CK(cudaGraphAddKernelNode(&nset, g, nullptr, 0, &kp));
        CK(cudaGraphAddNode(&ncond, g, &nset, 1, &p));
        cudaGraph_t body = p.conditional.phGraph_out[0];
        cudaStream_t cs;
        CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        CK(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < 30; ++i) k_big<<<148, 256, 0, cs>>>(nullptr, bg);
        k_dec<<<1, 1, 0, cs>>>(d, h);
        CK(cudaStreamEndCapture(cs, &body));
        cudaGraphExec_t ge;
        CK(cudaGraphInstantiate(&ge, g, 0));
        printf("WHILE body (10 iters x 31 kernels, 768-B params): %.3f us per kernel\n", time_graph(ge, s, 20) * 1e3 / 310);
    }
    // grid barrier cost
    unsigned* bar;
    CK(cudaMalloc(&bar, 8));
    CK(cudaMemset(bar, 0, 8));
    for (int threads : {256, 1024}) {
        for (int blocks : {148, 296}) {
            if (threads == 1024 && blocks == 296) continue;
            const int nb = 1000;
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            void* args[] = {&bar, (void*)&nb};
            CK(cudaLaunchCooperativeKernel((void*)k_barriers, dim3(blocks), dim3(threads), args, 0, s));
            CK(cudaStreamSynchronize(s));
            cudaEventRecord(a, s);
            CK(cudaLaunchCooperativeKernel((void*)k_barriers, dim3(blocks), dim3(threads), args, 0, s));
            cudaEventRecord(b, s);
            CK(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("grid barrier, %d CTAs x %d threads: %.3f us per barrier\n", blocks, threads, ms * 1e3 / nb);
        }
    }
    return 0;
}
