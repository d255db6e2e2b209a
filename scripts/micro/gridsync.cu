// Microbenchmark: cost of one cooperative-groups grid barrier on this GPU (k_rm's round structure).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gridsync scripts/micro/gridsync.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__global__ void k(int iters, unsigned* sink) {
    cg::grid_group g = cg::this_grid();
    unsigned acc = 0;
    for (int i = 0; i < iters; ++i) {
        acc += threadIdx.x ^ i;
        g.sync();
    }
    if (acc == 0xFFFFFFFF) sink[0] = acc;
}
int main() {
    unsigned* sink;
    cudaMalloc(&sink, 4);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bs : {256, 512, 1024}) {
        int per = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, bs, 0);
        for (int mult : {1, per}) {
            int grid = sms * mult, iters = 2000;
            void* args[] = {&iters, &sink};
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            cudaLaunchCooperativeKernel((void*)k, grid, bs, args, 0, 0);
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k, grid, bs, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            printf("block %d x grid %d: %.3f us per grid.sync\n", bs, grid, 1e3 * ms / iters);
        }
    }
    return 0;
}
