// Diagnostic: cost of cooperative_groups grid.sync() with one 256-thread CTA per SM, and
// whether a cooperative launch can be captured into a CUDA graph.
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__global__ void syncs(int reps, int* out) {
    cg::grid_group g = cg::this_grid();
    int acc = 0;
    for (int r = 0; r < reps; ++r) {
        acc += threadIdx.x;
        g.sync();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = acc;
}
int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int* o;
    cudaMalloc(&o, 4);
    cudaStream_t st;
    cudaStreamCreate(&st);
    for (int reps : {1, 1000}) {
        void* args[] = {&reps, &o};
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaLaunchCooperativeKernel((void*)syncs, sms, 256, args, 0, st);
        cudaEventRecord(a, st);
        cudaLaunchCooperativeKernel((void*)syncs, sms, 256, args, 0, st);
        cudaEventRecord(b, st);
        cudaStreamSynchronize(st);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("reps %d: %.2f us total, %.3f us per sync\n", reps, ms * 1e3, ms * 1e3 / reps);
    }
    // capture
    cudaGraph_t g;
    cudaGraphExec_t ge;
    int reps = 10;
    void* args[] = {&reps, &o};
    cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    cudaError_t e1 = cudaLaunchCooperativeKernel((void*)syncs, sms, 256, args, 0, st);
    cudaError_t e2 = cudaStreamEndCapture(st, &g);
    cudaError_t e3 = e2 == cudaSuccess ? cudaGraphInstantiate(&ge, g, 0) : e2;
    cudaError_t e4 = e3 == cudaSuccess ? cudaGraphLaunch(ge, st) : e3;
    cudaError_t e5 = cudaStreamSynchronize(st);
    printf("capture: launch %s end %s inst %s run %s sync %s\n", cudaGetErrorString(e1), cudaGetErrorString(e2),
           cudaGetErrorString(e3), cudaGetErrorString(e4), cudaGetErrorString(e5));
}
