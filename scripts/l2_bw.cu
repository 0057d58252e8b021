// Diagnostic: L2-resident and HBM read bandwidth on this B200 — the L2 roofline denominator of the
// bank-pass MAC (its filter rows come from L2) and a cross-check of the HBM figure. Reads a buffer
// of `mb` MB repeatedly with 16-byte L1-bypassing loads (ld.global.cg), U independent loads in
// flight per thread, from a grid of k CTAs per SM; GB/s = bytes read / time (best of 5, events).
// Prints one JSON object per (size, k, U) and a final summary line {"l2_read_gbs": ..., "hbm_read_gbs": ...}.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2_bw l2_bw.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int U>
__global__ void __launch_bounds__(256) read_kernel(const float4* __restrict__ p, size_t n4, int reps, float* sink) {
    float acc = 0.f;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    for (int r = 0; r < reps; ++r) {
        size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
        for (; i + (U - 1) * stride < n4; i += U * stride) {
            float4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) v[u] = __ldcg(p + i + u * stride);
#pragma unroll
            for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
        }
        for (; i < n4; i += stride) {
            const float4 v = __ldcg(p + i);
            acc += v.x + v.y + v.z + v.w;
        }
    }
    if (acc == 1234.5f) sink[0] = acc;
}

template <int U>
float run(const float4* p, size_t n4, int grid, int reps, float* sink) {
    read_kernel<U><<<grid, 256>>>(p, n4, 1, sink);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    for (int t = 0; t < 5; ++t) {
        cudaEventRecord(a);
        read_kernel<U><<<grid, 256>>>(p, n4, reps, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int main() {
    cudaDeviceProp prop;
    cudaGetDeviceProperties(&prop, 0);
    const size_t sizes_mb[] = {16, 32, 48, 64, 4096};
    float* sink;
    cudaMalloc(&sink, 4);
    double best_l2 = 0, best_hbm = 0;
    for (size_t mb : sizes_mb) {
        const size_t bytes = mb << 20;
        float4* p;
        if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
        cudaMemset(p, 0, bytes);
        const size_t n4 = bytes / 16;
        const int reps = mb >= 1024 ? 3 : (int)(16384 / mb);
        for (int per_sm : {4, 8}) {
            const int grid = prop.multiProcessorCount * per_sm;
            for (int U : {1, 4, 8}) {
                const float ms = U == 1 ? run<1>(p, n4, grid, reps, sink)
                                        : (U == 4 ? run<4>(p, n4, grid, reps, sink) : run<8>(p, n4, grid, reps, sink));
                const double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
                printf("{\"buffer_mb\": %zu, \"ctas_per_sm\": %d, \"threads\": 256, \"loads_in_flight\": %d, \"gbs\": %.1f}\n",
                       mb, per_sm, U, gbs);
                if (mb <= 64 && gbs > best_l2) best_l2 = gbs;
                if (mb >= 1024 && gbs > best_hbm) best_hbm = gbs;
            }
        }
        cudaFree(p);
    }
    printf("{\"l2_read_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"sms\": %d, \"l2_bytes\": %d}\n", best_l2, best_hbm,
           prop.multiProcessorCount, prop.l2CacheSize);
    return 0;
}
