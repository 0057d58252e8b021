// Diagnostic: L2-resident and HBM read bandwidth on this B200 (the roofline denominators for the
// bank kernels, whose filter traffic is served from L2). Reads a buffer of `mb` MB repeatedly with
// 16-byte __ldcg loads from a persistent grid (k CTAs per SM); reports GB/s = bytes read / time.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw l2_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512) read_kernel(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r) {
        for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

int main(int argc, char** argv) {
    int dev = 0;
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, dev);
    const size_t sizes_mb[] = {8, 16, 32, 48, 64, 96, 4096};
    float* sink;
    cudaMalloc(&sink, 4);
    for (size_t mb : sizes_mb) {
        size_t bytes = mb << 20;
        float4* p;
        if (cudaMalloc(&p, bytes) != cudaSuccess) { printf("alloc fail\n"); return 1; }
        cudaMemset(p, 0, bytes);
        size_t n4 = bytes / 16;
        int reps = mb >= 1024 ? 3 : (int)(8192 / mb);
        for (int per_sm : {2, 4}) {
            int grid = prop.multiProcessorCount * per_sm;
            read_kernel<<<grid, 512>>>(p, n4, 1, sink);
            cudaEvent_t a, b;
            cudaEventCreate(&a); cudaEventCreate(&b);
            float best = 1e30f;
            for (int t = 0; t < 5; ++t) {
                cudaEventRecord(a);
                read_kernel<<<grid, 512>>>(p, n4, reps, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms; cudaEventElapsedTime(&ms, a, b);
                if (ms < best) best = ms;
            }
            printf("{\"buffer_mb\": %zu, \"ctas_per_sm\": %d, \"gbs\": %.1f}\n", mb, per_sm,
                   (double)bytes * reps / (best * 1e-3) / 1e9);
        }
        cudaFree(p);
    }
    printf("{\"sms\": %d, \"l2_bytes\": %d}\n", prop.multiProcessorCount, prop.l2CacheSize);
    return 0;
}
