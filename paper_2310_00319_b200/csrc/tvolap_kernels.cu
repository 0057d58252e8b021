// TVOLAP hot-path kernels for sm_100a.
//
// The reference processes one hop per lane with scalar fp64 code
// (proj/src/engine.cpp:60-106). Here one fused kernel runs n_hops consecutive
// hops for all sources. Each source is owned by a cluster of P CTAs (thread
// block cluster, distributed shared memory); per hop every CTA
//   K1  frames the hop with the periodic Hann window and takes the 4L real
//       FFT as a pruned 2L-point complex Stockham FFT in shared memory
//       (engine.cpp:77-82, spectral.cpp:99-125),
//   K2  writes its 1/P slice of the packed spectrum into the HBM delay line,
//       two parity rings of depth M (ring[s][hop&1][(hop>>1) mod M]) —
//       equivalent to the reference's 2M-1 ring read at stride 2
//       (engine.hpp:41, engine.cpp:69-70,88),
//   K3  accumulates Y = sum_m H[m] (.) X_{hop-2m} over its bin slice with
//       coalesced 128-bit loads, M split over thread groups and reduced in smem
//       (engine.cpp:85-92, spectral.cpp:160-166),
//   K5  gathers the full Y from the cluster over DSMEM, takes the inverse real
//       FFT and does the hop-2 overlap-add with gain 1/2 for its 1/P share of
//       the output (spectral.cpp:127-158, engine.cpp:94-102).
// Lanes never wait on each other, so the kernel needs no grid-wide sync and
// state (input history, OLA accumulators) stays in shared memory across the
// hops of one launch.
//
// Spectra are stored packed: 2L complex64 per frame, bin 0 holding
// (Re X_0, Re X_2L) — both are exactly real (spectral.cpp:121-123) — so a frame
// is a whole number of float4s and the MAC treats bin 0 as two real products.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "tvolap_fft.cuh"
#include "tvolap_internal.cuh"
#include "workload.h"

namespace cg = cooperative_groups;

namespace tvb {
namespace {

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct SmemLayout {
    size_t tw, pk, win, x0, x1, fa, fb, red, yb, ola, total;
    __host__ __device__ SmemLayout(int L, int P, int E, int threads) {
        const size_t N = 2 * (size_t)L;
        tw = 0;
        pk = align16(tw + N * sizeof(float2));
        win = align16(pk + (N + 2) * sizeof(float2));
        x0 = align16(win + N * sizeof(float));
        x1 = align16(x0 + L * sizeof(float));
        fa = align16(x1 + L * sizeof(float));
        fb = align16(fa + N * sizeof(float2));
        red = align16(fb + N * sizeof(float2));
        yb = align16(red + (size_t)threads * E * sizeof(float4));
        ola = align16(yb + 2 * (size_t)E * (N / P) * sizeof(float2));
        total = align16(ola + (size_t)E * 3 * (L / P) * sizeof(float));
    }
};

__device__ __forceinline__ void cmac4(float4& acc, float& aux, const float4 h, const float4 x) {
    acc.x = fmaf(h.x, x.x, acc.x);
    acc.x = fmaf(-h.y, x.y, acc.x);
    acc.y = fmaf(h.x, x.y, acc.y);
    acc.y = fmaf(h.y, x.x, acc.y);
    acc.z = fmaf(h.z, x.z, acc.z);
    acc.z = fmaf(-h.w, x.w, acc.z);
    acc.w = fmaf(h.z, x.w, acc.w);
    acc.w = fmaf(h.w, x.z, acc.w);
    aux = fmaf(h.y, x.y, aux);  // Nyquist product, only kept for the packed bin 0
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
    return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

template <int E>
__global__ void __launch_bounds__(1024) tvolap_hop_kernel(const HopParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int L = p.L, N = 2 * L, M = p.M, P = p.P;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int s = blockIdx.x / P;
    const int r = blockIdx.x % P;  // == cluster rank (1-D clusters of P consecutive CTAs)
    const SmemLayout lay(L, P, E, NT);
    float2* s_tw = reinterpret_cast<float2*>(smem + lay.tw);
    float2* s_pk = reinterpret_cast<float2*>(smem + lay.pk);
    float* s_win = reinterpret_cast<float*>(smem + lay.win);
    float* xprev = reinterpret_cast<float*>(smem + lay.x0);
    float* xcur = reinterpret_cast<float*>(smem + lay.x1);
    float2* s_fa = reinterpret_cast<float2*>(smem + lay.fa);
    float2* s_fb = reinterpret_cast<float2*>(smem + lay.fb);
    float4* s_red = reinterpret_cast<float4*>(smem + lay.red);
    float2* s_yb = reinterpret_cast<float2*>(smem + lay.yb);
    float* s_ola = reinterpret_cast<float*>(smem + lay.ola);

    const int Np = N / P;   // packed bins owned by this CTA
    const int V = Np / 2;   // float4 per slice
    const int Lp = L / P;   // output samples owned by this CTA
    const int VT = V < NT ? V : NT;
    const int G = NT / VT;  // partition groups
    const int f0 = tid % VT, g = tid / VT;
    const long spec4 = N / 2;  // float4 per spectrum

    for (int i = tid; i < N; i += NT) {
        s_tw[i] = p.tw[i];
        s_win[i] = p.win[i];
    }
    for (int i = tid; i <= N; i += NT) s_pk[i] = p.pk[i];
    for (int i = tid; i < L; i += NT) xprev[i] = p.hist[(long)s * L + i];
    for (int i = tid; i < E * 3 * Lp; i += NT) {
        const int e = i / (3 * Lp), rem = i % (3 * Lp), j = rem / Lp, u = rem % Lp;
        s_ola[i] = p.ola[((long)s * E + e) * 3 * L + j * L + r * Lp + u];
    }
    __syncthreads();

    const float4* ring4 = reinterpret_cast<const float4*>(p.ring);
    const float4* pool4 = reinterpret_cast<const float4*>(p.pool);

    for (int k = 0; k < p.n_hops; ++k) {
        const long hop = p.hop0 + k;
        const int par = (int)(hop & 1);
        const int sl = (int)((hop >> 1) % M);

        // ---- K1: frame (previous hop | this hop) x Hann, zero-pad to 4L, FFT.
        const float* inp = p.in + (long)s * p.in_stride + (long)k * L;
        for (int i = tid; i < L; i += NT) xcur[i] = inp[i];
        __syncthreads();
        for (int j = tid; j < L; j += NT) {
            const int i0 = 2 * j, i1 = 2 * j + 1;
            const float a = (i0 < L ? xprev[i0] : xcur[i0 - L]) * s_win[i0];
            const float b = (i1 < L ? xprev[i1] : xcur[i1 - L]) * s_win[i1];
            s_fa[j] = make_float2(a, b);
        }
        __syncthreads();
        const float2* Z = fft_stockham<false>(s_fa, s_fb, N, s_tw, true, tid, NT);

        // ---- K2: this CTA's slice of X_hop into the delay line.
        float2* ringw = p.ring + (((long)s * 2 + par) * M + sl) * N + (long)r * Np;
        for (int kk = tid; kk < Np; kk += NT) ringw[kk] = untangle_packed(Z, N, r * Np + kk, s_pk);
        float* t = xprev;
        xprev = xcur;
        xcur = t;
        __syncthreads();

        // ---- K3: Y = sum_m H[m] X_{hop-2m} over the slice.
        const int entry = p.sched ? p.sched[(long)k * p.sched_stride + s] : p.entry_base + s;
        const float4* xb = ring4 + (((long)s * 2 + par) * M) * spec4 + (long)r * V;
        const float4* hb = pool4 + ((long)entry * E * M) * spec4 + (long)r * V;
        float2* yb = s_yb + (size_t)(k & 1) * E * Np;
        for (int fi = f0; fi < V; fi += VT) {
            float4 acc[E];
            float aux[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
                aux[e] = 0.f;
            }
            int m = g;
            int slot = ((sl - g) % M + M) % M;
            for (; m + 3 * G < M; m += 4 * G) {
                int s1 = slot - G;
                if (s1 < 0) s1 += M;
                int s2 = s1 - G;
                if (s2 < 0) s2 += M;
                int s3 = s2 - G;
                if (s3 < 0) s3 += M;
                const float4 x0 = __ldcg(xb + slot * spec4 + fi);
                const float4 x1 = __ldcg(xb + s1 * spec4 + fi);
                const float4 x2 = __ldcg(xb + s2 * spec4 + fi);
                const float4 x3 = __ldcg(xb + s3 * spec4 + fi);
                float4 h[E][4];
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const float4* he = hb + ((long)e * M + m) * spec4 + fi;
                    h[e][0] = __ldg(he);
                    h[e][1] = __ldg(he + G * spec4);
                    h[e][2] = __ldg(he + 2 * G * spec4);
                    h[e][3] = __ldg(he + 3 * G * spec4);
                }
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    cmac4(acc[e], aux[e], h[e][0], x0);
                    cmac4(acc[e], aux[e], h[e][1], x1);
                    cmac4(acc[e], aux[e], h[e][2], x2);
                    cmac4(acc[e], aux[e], h[e][3], x3);
                }
                slot = s3 - G;
                if (slot < 0) slot += M;
            }
            for (; m < M; m += G) {
                const float4 x0 = __ldcg(xb + slot * spec4 + fi);
#pragma unroll
                for (int e = 0; e < E; ++e) cmac4(acc[e], aux[e], __ldg(hb + ((long)e * M + m) * spec4 + fi), x0);
                slot -= G;
                if (slot < 0) slot += M;
            }
            if (r == 0 && fi == 0) {
#pragma unroll
                for (int e = 0; e < E; ++e) {  // packed bin 0: (H_0 X_0, H_N X_N) as two real products
                    acc[e].x += aux[e];
                    acc[e].y = aux[e];
                }
            }
            if (G == 1) {
#pragma unroll
                for (int e = 0; e < E; ++e) reinterpret_cast<float4*>(yb + (size_t)e * Np)[fi] = acc[e];
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) s_red[(g * VT + f0) * E + e] = acc[e];
            }
        }
        if (G > 1) {
            __syncthreads();
            for (int i = tid; i < VT * E; i += NT) {
                const int f = i / E, e = i % E;
                float4 sum = s_red[f * E + e];
                for (int gg = 1; gg < G; ++gg) sum = f4add(sum, s_red[(gg * VT + f) * E + e]);
                reinterpret_cast<float4*>(yb + (size_t)e * Np)[f] = sum;
            }
        }
        if (P > 1)
            cg::this_cluster().sync();
        else
            __syncthreads();

        // ---- K5: gather Y over DSMEM, inverse real FFT, hop-2 overlap-add.
        for (int e = 0; e < E; ++e) {
            for (int q = 0; q < P; ++q) {
                const float4* src = reinterpret_cast<const float4*>(yb + (size_t)e * Np);
                if (q != r) src = cg::this_cluster().map_shared_rank(src, q);
                float4* dst = reinterpret_cast<float4*>(s_fa + (size_t)q * Np);
                for (int i = tid; i < V; i += NT) dst[i] = src[i];
            }
            __syncthreads();
            for (int i = tid; i < N; i += NT) s_fb[i] = tangle_packed(s_fa, N, i, s_pk);
            __syncthreads();
            const float* yf = reinterpret_cast<const float*>(fft_stockham<true>(s_fb, s_fa, N, s_tw, false, tid, NT));
            const float sc = 1.0f / (float)N;
            float* A = s_ola + e * 3 * Lp;
            float* o = p.out + ((long)s * E + e) * p.out_stride + (long)k * L;
            for (int u = tid; u < Lp; u += NT) {
                const int ug = r * Lp + u;
                const float y0 = yf[ug] * sc, y1 = yf[L + ug] * sc, y2 = yf[2 * L + ug] * sc,
                            y3 = yf[3 * L + ug] * sc;
                o[ug] = 0.5f * (y0 + A[u]);
                A[u] = y1 + A[Lp + u];
                A[Lp + u] = y2 + A[2 * Lp + u];
                A[2 * Lp + u] = y3;
            }
            __syncthreads();
        }
    }
    if (P > 1) cg::this_cluster().sync();  // no CTA leaves while a peer may still read its Y slice

    if (r == 0)
        for (int i = tid; i < L; i += NT) p.hist[(long)s * L + i] = xprev[i];
    for (int i = tid; i < E * 3 * Lp; i += NT) {
        const int e = i / (3 * Lp), rem = i % (3 * Lp), j = rem / Lp, u = rem % Lp;
        p.ola[((long)s * E + e) * 3 * L + j * L + r * Lp + u] = s_ola[i];
    }
}

// K4: transform IR slices into packed partition spectra (partition.cpp:20-51).
__global__ void __launch_bounds__(256) partition_kernel(int L, int M, long rows, const float* __restrict__ ir,
                                                        long ir_stride, long ir_len, float2* __restrict__ pool,
                                                        long row0, const float2* __restrict__ tw,
                                                        const float2* __restrict__ pk) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int N = 2 * L, tid = threadIdx.x, NT = blockDim.x;
    float2* s_tw = reinterpret_cast<float2*>(smem);
    float2* s_pk = s_tw + N;
    float2* s_fa = s_pk + N + 2;
    float2* s_fb = s_fa + N;
    for (int i = tid; i < N; i += NT) s_tw[i] = tw[i];
    for (int i = tid; i <= N; i += NT) s_pk[i] = pk[i];
    __syncthreads();
    const long tasks = rows * M;
    for (long task = blockIdx.x; task < tasks; task += gridDim.x) {
        const long row = task / M;
        const int m = (int)(task % M);
        const float* h = ir + row * ir_stride;
        const long base = (long)m * N;
        for (int j = tid; j < L; j += NT) {
            const long i0 = base + 2 * j;
            const float a = i0 < ir_len ? h[i0] : 0.f;
            const float b = i0 + 1 < ir_len ? h[i0 + 1] : 0.f;
            s_fa[j] = make_float2(a, b);
        }
        __syncthreads();
        const float2* Z = fft_stockham<false>(s_fa, s_fb, N, s_tw, true, tid, NT);
        float2* outp = pool + ((row0 + row) * M + m) * N;
        for (int kk = tid; kk < N; kk += NT) outp[kk] = untangle_packed(Z, N, kk, s_pk);
        __syncthreads();
    }
}

// forward_real on a batch (spectral.cpp:99-125): full real input of n = 2N samples.
__global__ void forward_real_kernel(int N, const float* __restrict__ x, float2* __restrict__ bins,
                                    const float2* __restrict__ tw, const float2* __restrict__ pk) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, NT = blockDim.x;
    float2* s_fa = reinterpret_cast<float2*>(smem);
    float2* s_fb = s_fa + N;
    const float* xb = x + (long)blockIdx.x * 2 * N;
    for (int j = tid; j < N; j += NT) s_fa[j] = make_float2(xb[2 * j], xb[2 * j + 1]);
    __syncthreads();
    const float2* Z = fft_stockham<false>(s_fa, s_fb, N, tw, false, tid, NT);
    float2* out = bins + (long)blockIdx.x * (N + 1);
    for (int k = tid; k <= N; k += NT) {
        float2 v = untangle(Z, N, k, pk);
        if (k == 0 || k == N) v.y = 0.f;
        out[k] = v;
    }
}

// inverse_real on a batch (spectral.cpp:127-158).
__global__ void inverse_real_kernel(int N, const float2* __restrict__ bins, float* __restrict__ x,
                                    const float2* __restrict__ tw, const float2* __restrict__ pk) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int tid = threadIdx.x, NT = blockDim.x;
    float2* s_fa = reinterpret_cast<float2*>(smem);
    float2* s_fb = s_fa + N;
    const float2* b = bins + (long)blockIdx.x * (N + 1);
    for (int k = tid; k < N; k += NT) {
        const float2 xk = b[k];
        const float2 t = b[N - k];
        const float2 xm = make_float2(t.x, -t.y);
        const float2 even = make_float2(0.5f * (xk.x + xm.x), 0.5f * (xk.y + xm.y));
        const float2 odd = cmulc(make_float2(0.5f * (xk.x - xm.x), 0.5f * (xk.y - xm.y)), pk[k]);
        s_fa[k] = make_float2(even.x - odd.y, even.y + odd.x);
    }
    __syncthreads();
    const float2* z = fft_stockham<true>(s_fa, s_fb, N, tw, false, tid, NT);
    const float sc = 1.0f / (float)N;
    float* xo = x + (long)blockIdx.x * 2 * N;
    for (int j = tid; j < N; j += NT) {
        xo[2 * j] = z[j].x * sc;
        xo[2 * j + 1] = z[j].y * sc;
    }
}

__global__ void mac_kernel(long n, const float2* __restrict__ acc, const float2* __restrict__ a,
                           const float2* __restrict__ b, float2* __restrict__ out) {
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < n; i += (long)gridDim.x * blockDim.x) {
        const float2 c = acc[i], x = a[i], y = b[i];
        out[i] = make_float2(c.x + (x.x * y.x - x.y * y.y), c.y + (x.x * y.y + x.y * y.x));
    }
}

__global__ void gen_white_kernel(uint64_t seed, long lane0, long lanes, long t0, long n, float* out, long stride) {
    const long total = lanes * n;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long l = i / n, t = i % n;
        out[l * stride + t] =
            (float)tv_uniform_pm1(tv_rand64(seed, tv_stream_input((uint64_t)(lane0 + l)), (uint64_t)(t0 + t)));
    }
}

__global__ void __launch_bounds__(256) gen_irs_kernel(uint64_t seed, const long* lanes, const long* ears,
                                                      const long* ks, const double* t60, double fs, long len,
                                                      float* out) {
    __shared__ double red[256];
    const long i = blockIdx.x;
    const uint64_t st = tv_stream_ir((uint64_t)lanes[i], (uint64_t)ears[i], (uint64_t)ks[i]);
    const double T = t60[i];
    double e = 0.0;
    for (long n = threadIdx.x; n < len; n += blockDim.x) {
        const double h = tv_ir_tap(seed, st, (uint64_t)n, T, fs);
        e += h * h;
    }
    red[threadIdx.x] = e;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    const double g = red[0] > 0.0 ? 1.0 / sqrt(red[0]) : 0.0;
    for (long n = threadIdx.x; n < len; n += blockDim.x)
        out[i * len + n] = (float)(tv_ir_tap(seed, st, (uint64_t)n, T, fs) * g);
}

__global__ void mix_kernel(long sources, long ears, long samples, const float* __restrict__ out, long out_stride,
                           float* __restrict__ mix, long mix_stride) {
    const long total = ears * samples;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long e = i / samples, t = i % samples;
        float acc = 0.f;
        for (long s = 0; s < sources; ++s) acc += out[(s * ears + e) * out_stride + t];
        mix[e * mix_stride + t] = acc;
    }
}

int grid_for(long work, int threads) {
    long b = (work + threads - 1) / threads;
    return (int)std::max<long>(1, std::min<long>(b, 148L * 16));
}

int fft_threads(int N) { return std::max(32, std::min(256, N / 4)); }

}  // namespace

size_t hop_kernel_smem_bytes(int L, int P, int E, int threads) { return SmemLayout(L, P, E, threads).total; }

cudaError_t launch_hop_kernel(const HopParams& p, int E, int threads, cudaStream_t stream) {
    const size_t smem = hop_kernel_smem_bytes(p.L, p.P, E, threads);
    void (*fn)(const HopParams) = E == 2 ? tvolap_hop_kernel<2> : tvolap_hop_kernel<1>;
    cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    if (p.P > 1) {
        err = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (err != cudaSuccess) return err;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(p.S * p.P));
    cfg.blockDim = dim3((unsigned)threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)p.P;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = p.P > 1 ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, fn, p);
}

cudaError_t launch_partition(int L, int M, long rows, const float* ir, long ir_stride, long ir_len, float2* pool,
                             long row0, const float2* tw, const float2* pk, cudaStream_t stream) {
    const int N = 2 * L;
    const int threads = fft_threads(N);
    const size_t smem = (size_t)(4 * N + 2) * sizeof(float2);
    cudaError_t err = cudaFuncSetAttribute(partition_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const long tasks = rows * M;
    const int grid = (int)std::max<long>(1, std::min<long>(tasks, 148L * 8));
    partition_kernel<<<grid, threads, smem, stream>>>(L, M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk);
    return cudaGetLastError();
}

cudaError_t launch_forward_real(long n, long batch, const float* x, float2* bins, const float2* tw,
                                const float2* pk, cudaStream_t stream) {
    const int N = (int)(n / 2);
    const size_t smem = 2 * (size_t)N * sizeof(float2);
    cudaError_t err =
        cudaFuncSetAttribute(forward_real_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    forward_real_kernel<<<(unsigned)batch, fft_threads(N), smem, stream>>>(N, x, bins, tw, pk);
    return cudaGetLastError();
}

cudaError_t launch_inverse_real(long n, long batch, const float2* bins, float* x, const float2* tw,
                                const float2* pk, cudaStream_t stream) {
    const int N = (int)(n / 2);
    const size_t smem = 2 * (size_t)N * sizeof(float2);
    cudaError_t err =
        cudaFuncSetAttribute(inverse_real_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    inverse_real_kernel<<<(unsigned)batch, fft_threads(N), smem, stream>>>(N, bins, x, tw, pk);
    return cudaGetLastError();
}

cudaError_t launch_mac(long nbins, long batch, const float2* acc, const float2* a, const float2* b, float2* out,
                       cudaStream_t stream) {
    const long n = nbins * batch;
    mac_kernel<<<grid_for(n, 256), 256, 0, stream>>>(n, acc, a, b, out);
    return cudaGetLastError();
}

cudaError_t launch_gen_white(uint64_t seed, long lane0, long lanes, long t0, long n, float* out, long stride,
                             cudaStream_t stream) {
    gen_white_kernel<<<grid_for(lanes * n, 256), 256, 0, stream>>>(seed, lane0, lanes, t0, n, out, stride);
    return cudaGetLastError();
}

cudaError_t launch_gen_irs(uint64_t seed, long count, const long* lanes, const long* ears, const long* ks,
                           const double* t60, double fs, long len, float* out, cudaStream_t stream) {
    if (count <= 0) return cudaSuccess;
    gen_irs_kernel<<<(unsigned)count, 256, 0, stream>>>(seed, lanes, ears, ks, t60, fs, len, out);
    return cudaGetLastError();
}

cudaError_t launch_mix(long sources, long ears, long samples, const float* out, long out_stride, float* mix,
                       long mix_stride, cudaStream_t stream) {
    mix_kernel<<<grid_for(ears * samples, 256), 256, 0, stream>>>(sources, ears, samples, out, out_stride, mix,
                                                                 mix_stride);
    return cudaGetLastError();
}

}  // namespace tvb
