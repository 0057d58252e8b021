// TVOLAP hot-path kernels for sm_100a.
//
// The reference processes one hop per lane with scalar fp64 code
// (proj/src/engine.cpp:60-106). Here each source (lane) is owned by a thread
// block cluster of P CTAs (distributed shared memory); every CTA owns 1/P of
// the spectrum bins and 1/P of the output samples. Per hop:
//   K1  frame the hop with the periodic Hann window and take the 4L real FFT as
//       a pruned 2L-point complex Stockham FFT in shared memory
//       (engine.cpp:77-82, spectral.cpp:99-125),
//   K2  write the packed spectrum into the HBM delay line: two parity rings of
//       D = M + 8 slots (ring[s][hop&1][(hop>>1) mod D]) — equivalent to the
//       reference's 2M-1 ring read at stride 2 (engine.hpp:41, engine.cpp:69-70,88),
//   K3  accumulate Y = sum_m H[m] (.) X_{hop-2m} over the bin slice with
//       coalesced 128-bit loads, partitions in contiguous groups reduced in smem
//       (engine.cpp:85-92, spectral.cpp:160-166),
//   K5  gather Y over DSMEM, inverse real FFT, hop-2 overlap-add with gain 1/2
//       (spectral.cpp:127-158, engine.cpp:94-102).
// tvolap_hop_kernel runs one hop at a time (process(), the latency path);
// tvolap_block_kernel runs blocks of J hops with the delay-line / filter slices
// shared across the block's hops (process_hops(), the throughput path). Both
// use the same operations in the same order, so their outputs are bit-identical.
// partition_kernel is K4 (partition.cpp:20-51) for staged filter sets.
// Lanes never wait on each other: no grid-wide sync; history and OLA state stay
// in shared memory across the hops of a launch.
//
// Spectra are stored packed: 2L complex64 per frame, bin 0 holding
// (Re X_0, Re X_2L) — both are exactly real (spectral.cpp:121-123) — so a frame
// is a whole number of float4s and the MAC treats bin 0 as two real products.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "tvolap_fft.cuh"
#include "tvolap_internal.cuh"
#include "workload.h"

namespace cg = cooperative_groups;

#ifdef TVOLAP_PHASE_PROF
// Diagnostic build only (scripts/phase_prof.py): SM cycles per block-kernel phase, summed over
// CTAs (thread 0 of each CTA), read back with tvolap_phase_counters().
__device__ unsigned long long g_phase[16];
#define PHASE_MARK(k)                                          \
    do {                                                       \
        if (threadIdx.x == 0) {                                \
            const long long t_ = clock64();                    \
            atomicAdd(&g_phase[k], (unsigned long long)(t_ - ph_t)); \
            ph_t = t_;                                         \
        }                                                      \
    } while (0)
#define PHASE_START() long long ph_t = clock64()
// launch timeline (globaltimer ns): [kind][launch][begin of CTA 0, end of the last CTA]
__device__ unsigned long long g_tl[2][4096][2];
__device__ unsigned g_tl_n[2], g_tl_done[2];
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define TL_BEGIN(kind)                                                               \
    do {                                                                             \
        if (threadIdx.x == 0 && blockIdx.x == 0) g_tl[kind][g_tl_n[kind] & 4095][0] = gtimer(); \
    } while (0)
#define TL_END(kind)                                                                 \
    do {                                                                             \
        __syncthreads();                                                             \
        if (threadIdx.x == 0) {                                                      \
            __threadfence();                                                         \
            if (atomicAdd(&g_tl_done[kind], 1u) == gridDim.x - 1) {                  \
                const unsigned n_ = g_tl_n[kind];                                    \
                g_tl[kind][n_ & 4095][1] = gtimer();                                 \
                g_tl_done[kind] = 0;                                                 \
                __threadfence();                                                     \
                g_tl_n[kind] = n_ + 1;                                               \
            }                                                                        \
        }                                                                            \
    } while (0)
#else
#define TL_BEGIN(kind) \
    do {               \
    } while (0)
#define TL_END(kind) \
    do {             \
    } while (0)
#define PHASE_MARK(k) \
    do {              \
    } while (0)
#define PHASE_START() \
    do {              \
    } while (0)
#endif

namespace tvb {

// process-wide launch knobs (tvolap_set_default_tuning "pdl", "k4_warp", "k4_prefetch")
long g_launch_pdl = 1;
long g_launch_k4_warp = 1;
long g_launch_k4_prefetch = 1;

namespace {

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

struct SmemLayout {
    size_t tw, pk, win, x0, x1, fa, fb, red, yb, ola, total;
    __host__ __device__ SmemLayout(int L, int P, int E, int qm) {
        const size_t N = 2 * (size_t)L;
        tw = 0;
        pk = align16(tw + N * sizeof(float2));
        win = align16(pk + (N + 2) * sizeof(float2));
        x0 = align16(win + N * sizeof(float));
        x1 = align16(x0 + L * sizeof(float));
        fa = align16(x1 + L * sizeof(float));
        fb = align16(fa + N * sizeof(float2));
        red = align16(fb + N * sizeof(float2));
        yb = align16(red + (qm > 1 ? (size_t)qm * (L / P) * E * sizeof(float4) : 0));
        ola = align16(yb + 2 * (size_t)E * (N / P) * sizeof(float2));
        total = align16(ola + (size_t)E * 3 * (L / P) * sizeof(float));
    }
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(src));
}

// TMA-engine bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, multiple of 16 bytes).
__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}
// bank per-output MAC: rows per L2 prefetch and prefetch distance (partitions ahead)
constexpr int kPfRows = 8;
constexpr int kPfDist = 2 * kPfRows;


// K4 fused into the hop kernels: at the start of the launch that latches a staged
// filter set, each cluster transforms its own source's new IR (partition.cpp:20-51):
// CTA r of the cluster takes partitions m = r, r+P, ..., `cap` of them per batched
// FFT, and writes the whole packed spectrum of each into the pool entry the MAC of
// this launch reads. The caller synchronises the cluster before the MAC.
template <int NC>
__device__ void fused_partition(const HopParams& p, int s, int r, int P, float2* fa, float2* fb, int cap,
                                size_t avail, const float2* tw, const float2* pk, int tid, int NT) {
    const int L = NC ? NC / 2 : p.L, N = 2 * L, M = p.M;
    const float* h = p.new_ir + (long)s * p.new_ir_stride;
    float2* dst = p.pool_w + ((long)(p.new_entry_base + s) * M) * N;
    if constexpr (NC != 0 && NC <= 1024) {
        // one warp per partition (as partition_warp_kernel, bit-identical), warp-private buffers
        // carved from the `avail` bytes at fa; partitions m = r, r + P, ... of this CTA
        // two partitions per warp in lockstep when the buffers allow (independent FFT chains)
        const int slots = (int)(avail / (NC * sizeof(float2)));
        const int warp = tid >> 5, lane = tid & 31;
        const bool vec = (p.new_ir_stride & 1) == 0 && (reinterpret_cast<uintptr_t>(p.new_ir) & 7) == 0;
        auto loader = [&](int m) {
            return [&, m](int, int n) -> float2 {
                const long i0 = (long)m * NC + 2 * n;
                if (m >= M) return make_float2(0.f, 0.f);
                if (vec && i0 + 1 < p.new_ir_len) return __ldcs(reinterpret_cast<const float2*>(h + i0));
                return make_float2(i0 < p.new_ir_len ? h[i0] : 0.f, i0 + 1 < p.new_ir_len ? h[i0 + 1] : 0.f);
            };
        };
        auto store = [&](const float2* buf, int m) { untangle_pairs_warp(buf, NC, pk, dst + (long)m * NC, lane); };
        if (slots >= 2 * (NT >> 5) && NC <= 512) {
            float2* buf = fa + (size_t)warp * 2 * NC;
            const int nw = NT >> 5;
            for (int m = r + warp * P; m < M; m += 2 * nw * P) {
                const int m2 = m + nw * P;  // second partition of this warp (may be past M)
                auto l0 = loader(m), l1 = loader(m2);
                auto load2 = [&](int t, int n) -> float2 { return t ? l1(t, n) : l0(t, n); };
                fft_warp4<false, NC, true, 2>(buf, p.tw + NC, lane, load2);
                store(buf, m);
                if (m2 < M) store(buf + NC, m2);
                __syncwarp();
            }
        } else {
            const int wfit = min(NT >> 5, slots);
            if (warp < wfit) {
                float2* buf = fa + (size_t)warp * NC;
                for (int m = r + warp * P; m < M; m += wfit * P) {
                    fft_warp4<false, NC, true>(buf, p.tw + NC, lane, loader(m));
                    store(buf, m);
                    __syncwarp();
                }
            }
        }
        __syncthreads();
        return;
    }
    const int nm = r < M ? (M - r + P - 1) / P : 0;
    const int lgL = 31 - __clz(L);
    for (int i0 = 0; i0 < nm; i0 += cap) {
        const int nt = min(cap, nm - i0);
        for (int i = tid; i < nt * L; i += NT) {
            const int f = i >> lgL, j = i & (L - 1);
            const long idx = (long)(r + (i0 + f) * P) * N + 2 * j;
            fa[(size_t)f * N + j] =
                make_float2(idx < p.new_ir_len ? h[idx] : 0.f, idx + 1 < p.new_ir_len ? h[idx + 1] : 0.f);
        }
        __syncthreads();
        const float2* Z = fft_batch<false, NC>(fa, fb, N, nt, tw, true, tid, NT);
        for (int f = 0; f < nt; ++f)
            untangle_store<NC>(Z + (size_t)f * N, N, pk, dst + (long)(r + (i0 + f) * P) * N, tid, NT);
        __syncthreads();
    }
}

template <int E, int NC>
__global__ void __launch_bounds__(1024) tvolap_hop_kernel(const HopParams p) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int L = NC ? NC / 2 : p.L, N = 2 * L, M = p.M, D = p.D, P = p.P;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int s = p.order ? p.order[blockIdx.x / P] : blockIdx.x / P;
    const int r = blockIdx.x % P;  // == cluster rank (1-D clusters of P consecutive CTAs)
    const SmemLayout lay(L, P, E, p.qm);
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
    // Partition groups: G = p.qm contiguous ranges [g M / G, (g+1) M / G), summed in g order —
    // the same grouping as the hop-blocked kernel, so both produce bit-identical outputs.
    const int G = p.qm;
    const int VT = max(1, min(V, NT / G));  // threads per group (each strides over the slice)
    const bool mac_thread = tid < G * VT;
    const int f0 = tid % VT, g = tid / VT;
    const int m0 = (int)((long)g * M / G), m1 = (int)((long)(g + 1) * M / G);
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
    if (p.new_ir) {  // latch a staged filter set: transform it here (K4), then the whole cluster sees it
        fused_partition<NC>(p, s, r, P, s_fa, s_fb, 1, lay.red - lay.fa, s_tw, s_pk, tid, NT);
        if (P > 1)
            cg::this_cluster().sync();
        else
            __syncthreads();
    }

    const float4* ring4 = reinterpret_cast<const float4*>(p.ring);
    const float4* pool4 = reinterpret_cast<const float4*>(p.pool);

    for (int k = 0; k < p.n_hops; ++k) {
        const long hop = p.hop0 + k;
        const int par = (int)(hop & 1);
        const int sl = (int)((hop >> 1) % D);

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
        const float2* Z = fft_stockham<false, NC>(s_fa, s_fb, N, s_tw, true, tid, NT);

        // ---- K2: this CTA's slice of X_hop into the delay line.
        float2* ringw = p.ring + (((long)s * 2 + par) * D + sl) * N + (long)r * Np;
        for (int kk = tid; kk < Np; kk += NT) ringw[kk] = untangle_packed(Z, N, r * Np + kk, s_pk);
        float* t = xprev;
        xprev = xcur;
        xcur = t;
        __syncthreads();

        // ---- K3: Y = sum_m H[m] X_{hop-2m} over the slice.
        const int entry = p.sched ? p.sched[(long)k * p.sched_stride + s] : p.entry_base + s;
        const float4* xb = ring4 + (((long)s * 2 + par) * D) * spec4 + (long)r * V;
        const float4* hb = pool4 + ((long)entry * E * M) * spec4 + (long)r * V;
        float2* yb = s_yb + (size_t)(k & 1) * E * Np;
        for (int fi = f0; mac_thread && fi < V; fi += VT) {
            float4 acc[E];
            float aux[E];
#pragma unroll
            for (int e = 0; e < E; ++e) {
                acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
                aux[e] = 0.f;
            }
            int slot = ((sl - m0) % D + D) % D;  // X_{hop-2m}: slot decrements with m
            int m = m0;
            for (; m + 4 <= m1; m += 4) {
                float4 x[4];
                float4 h[E][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    x[u] = __ldcg(xb + slot * spec4 + fi);
                    slot = slot == 0 ? D - 1 : slot - 1;
#pragma unroll
                    for (int e = 0; e < E; ++e) h[e][u] = __ldcg(hb + ((long)e * M + m + u) * spec4 + fi);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u)
#pragma unroll
                    for (int e = 0; e < E; ++e) cmac4(acc[e], aux[e], h[e][u], x[u]);
            }
            for (; m < m1; ++m) {
                const float4 x0 = __ldcg(xb + slot * spec4 + fi);
                slot = slot == 0 ? D - 1 : slot - 1;
#pragma unroll
                for (int e = 0; e < E; ++e) cmac4(acc[e], aux[e], __ldcg(hb + ((long)e * M + m) * spec4 + fi), x0);
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
                for (int e = 0; e < E; ++e) s_red[((size_t)g * V + fi) * E + e] = acc[e];
            }
        }
        if (G > 1) {
            __syncthreads();
            for (int i = tid; i < V * E; i += NT) {
                const int f = i / E, e = i % E;
                float4 sum = s_red[(size_t)f * E + e];
                for (int gg = 1; gg < G; ++gg) sum = f4add(sum, s_red[((size_t)gg * V + f) * E + e]);
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
            const float* yf = reinterpret_cast<const float*>(fft_stockham<true, NC>(s_fb, s_fa, N, s_tw, false, tid, NT));
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

// ============================================================================
// Streaming kernel with a bulk-copy ring (bank engines, one hop per call, P = 1): persistent CTAs
// (one per SM) walk the sources in the launch order, and the delay-line rows and filter rows of
// the MAC arrive in shared memory by cp.async.bulk (TMA) signalled on mbarriers — a ring of ST
// stages, each R partition steps of every partition group, refilled by one thread as soon as a
// stage is consumed and running ahead ACROSS sources, so the HBM stream does not stop while a
// source's transforms (K1, K5) run and bytes in flight are not tied to registers or to resident
// warps. The hop's own spectrum (partition 0) never travels through memory: K2 writes it into
// the stage's row next to the global delay-line store. Same partition groups and summation order
// as tvolap_hop_kernel: bit-identical outputs (spectral.cpp:160-166, engine.cpp:60-106).
constexpr int kRingSources = 64;  // sources per CTA whose (index, bank entry) the kernel tabulates up front
struct RingLayout {
    size_t tw, pk, win, x0, x1, fa, fb, red, yb, bar, tab, ring, stage, total;
    int G, R, ST;
    __host__ __device__ RingLayout(int L, int E, int G_, int R_, int ST_) : G(G_), R(R_), ST(ST_) {
        const size_t N = 2 * (size_t)L;
        tw = 0;
        pk = align16(tw + N * sizeof(float2));
        win = align16(pk + (N + 2) * sizeof(float2));
        x0 = align16(win + N * sizeof(float));
        x1 = align16(x0 + L * sizeof(float));
        fa = align16(x1 + L * sizeof(float));
        fb = align16(fa + N * sizeof(float2));
        red = align16(fb + N * sizeof(float2));
        yb = align16(red + (size_t)G * L * E * sizeof(float4));
        bar = align16(yb + (size_t)E * N * sizeof(float2));
        tab = align16(bar + 8 * 8);
        ring = (tab + 2 * kRingSources * sizeof(int) + 127) / 128 * 128;
        stage = (size_t)G * (1 + E) * R * N * sizeof(float2);
        total = ring + (size_t)ST * stage;
    }
};

__device__ __forceinline__ void ring_bar_init(unsigned bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void ring_bar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "RWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra RWAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void ring_expect(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void ring_copy(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

template <int E, int NC, int R, int ST>
__global__ void __launch_bounds__(1024) tvolap_hop_ring_kernel(const HopParams p) {
    extern __shared__ __align__(128) unsigned char smem[];
    constexpr int N = NC, L = NC / 2, V = L;
    const int M = p.M, D = p.D, G = p.qm;
    const int tid = threadIdx.x, NT = blockDim.x;  // NT == G * V: one float4 column of one group per thread
    const RingLayout lay(L, E, G, R, ST);
    float2* s_tw = reinterpret_cast<float2*>(smem + lay.tw);
    float2* s_pk = reinterpret_cast<float2*>(smem + lay.pk);
    float* s_win = reinterpret_cast<float*>(smem + lay.win);
    float* xprev = reinterpret_cast<float*>(smem + lay.x0);
    float* xcur = reinterpret_cast<float*>(smem + lay.x1);
    float2* s_fa = reinterpret_cast<float2*>(smem + lay.fa);
    float2* s_fb = reinterpret_cast<float2*>(smem + lay.fb);
    float4* s_red = reinterpret_cast<float4*>(smem + lay.red);
    float2* s_yb = reinterpret_cast<float2*>(smem + lay.yb);
    unsigned char* s_ring = smem + lay.ring;
    const unsigned bar0 = (unsigned)__cvta_generic_to_shared(smem + lay.bar);
    const unsigned ring0 = (unsigned)__cvta_generic_to_shared(s_ring);
    const unsigned rowB = N * sizeof(float2);              // one spectrum
    const unsigned blkB = R * rowB;                          // R rows of one kind
    const unsigned grpB = (1 + E) * blkB;                    // one group's X block + E filter blocks
    const unsigned stageB = (unsigned)lay.stage;
    const int MG = M / G, SPS = MG / R;                      // steps per group, stages per source (host-checked)
    const int f0 = tid % V, g = tid / V;
    const long hop = p.hop0;
    const int par = (int)(hop & 1), sl = (int)((hop >> 1) % D);
    const int nsrc = (p.S - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // sources of this CTA

    for (int i = tid; i < N; i += NT) {
        s_tw[i] = p.tw[i];
        s_win[i] = p.win[i];
    }
    for (int i = tid; i <= N; i += NT) s_pk[i] = p.pk[i];
    // this CTA's sources and their bank entries (the issuing thread must not chase them through
    // global memory in front of every stage)
    int* s_src = reinterpret_cast<int*>(smem + lay.tab);
    int* s_ent = s_src + kRingSources;
    for (int k = tid; k < nsrc; k += NT) {
        const int idx = (int)blockIdx.x + k * (int)gridDim.x;
        const int s = p.order ? p.order[idx] : idx;
        s_src[k] = s;
        s_ent[k] = p.sched[s];
    }
    if (tid == 0) {
        for (int b = 0; b < ST; ++b) ring_bar_init(bar0 + 8 * b);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();

    // stage j of this CTA's stream: source iteration j / SPS, steps t R .. t R + R - 1 of every group.
    // Issued by warp 0: lane 0 arms the stage's barrier with the byte count, then every lane issues
    // one of the stage's bulk copies (per group: the X block in up to two pieces around the
    // delay line's wrap, and E filter blocks).
    auto issue = [&](int j) {
        const int k = j / SPS, t = j - k * SPS;
        if (k >= nsrc) return;
        const int s = s_src[k], entry = s_ent[k];
        const int b = j % ST;
        const unsigned bar = bar0 + 8 * b, dst0 = ring0 + b * stageB;
        const int lane = tid & 31;
        if (lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // the stage's generic reads are done
            ring_expect(bar, G * grpB - (t == 0 ? rowB : 0));
        }
        __syncwarp();
        const float2* xbase = p.ring + (((long)s * 2 + par) * D) * N;
        for (int c = lane; c < G * (2 + E); c += 32) {
            const int gg = c / (2 + E), kind = c - gg * (2 + E);
            const int m = gg * MG + t * R;
            const unsigned dg = dst0 + gg * grpB;
            if (kind < 2) {
                // X rows: position q of the block holds slot (sl - m - (R - 1) + q) mod D, i.e. step r = R - 1 - q;
                // the hop's own spectrum (m = 0: q = R - 1 of group 0) comes from K2, not from memory
                const int cnt = R - ((gg == 0 && t == 0) ? 1 : 0);
                int lo = (sl - m - (R - 1)) % D;
                if (lo < 0) lo += D;
                const int first = min(cnt, D - lo);
                if (kind == 0) {
                    if (first > 0) ring_copy(dg, xbase + (long)lo * N, first * rowB, bar);
                } else if (first < cnt) {
                    ring_copy(dg + first * rowB, xbase, (cnt - first) * rowB, bar);
                }
            } else {
                const int e = kind - 2;
                ring_copy(dg + (1 + e) * blkB, p.pool + (((long)entry * E + e) * M + m) * N, blkB, bar);
            }
        }
    };
    if (tid < 32)
        for (int j = 0; j < ST; ++j) issue(j);

    for (int k = 0; k < nsrc; ++k) {
        const int s = s_src[k];
        const int jbase = k * SPS;

        // ---- K1: frame (previous hop | this hop) x Hann, zero-pad to 4L, FFT.
        const float* inp = p.in + (long)s * p.in_stride;
        for (int i = tid; i < L; i += NT) {
            xprev[i] = p.hist[(long)s * L + i];
            xcur[i] = inp[i];
        }
        __syncthreads();
        for (int j = tid; j < L; j += NT) {
            const int i0 = 2 * j, i1 = 2 * j + 1;
            const float a = (i0 < L ? xprev[i0] : xcur[i0 - L]) * s_win[i0];
            const float b = (i1 < L ? xprev[i1] : xcur[i1 - L]) * s_win[i1];
            s_fa[j] = make_float2(a, b);
        }
        for (int i = tid; i < L; i += NT) p.hist[(long)s * L + i] = xcur[i];
        __syncthreads();
        const float2* Z = fft_stockham<false, NC>(s_fa, s_fb, N, s_tw, true, tid, NT);

        // ---- K2: X_hop into the delay line and into the ring stage that holds step 0.
        {
            float2* ringw = p.ring + (((long)s * 2 + par) * D + sl) * N;
            float2* fresh = reinterpret_cast<float2*>(s_ring + (size_t)(jbase % ST) * stageB + (size_t)(R - 1) * rowB);
            for (int kk = tid; kk < N; kk += NT) {
                const float2 x = untangle_packed(Z, N, kk, s_pk);
                ringw[kk] = x;
                fresh[kk] = x;
            }
        }
        __syncthreads();

        // ---- K3: Y = sum_m H[m] X_{hop-2m}; thread (g, f0) walks its group's steps in order.
        float4 acc[E];
        float aux[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            acc[e] = make_float4(0.f, 0.f, 0.f, 0.f);
            aux[e] = 0.f;
        }
        for (int t = 0; t < SPS; ++t) {
            const int j = jbase + t, b = j % ST;
            ring_bar_wait(bar0 + 8 * b, (unsigned)((j / ST) & 1));
            const float4* xb = reinterpret_cast<const float4*>(s_ring + (size_t)b * stageB + (size_t)g * grpB) + f0;
#pragma unroll
            for (int r = 0; r < R; ++r) {
                const float4 x = xb[(R - 1 - r) * V];
#pragma unroll
                for (int e = 0; e < E; ++e) cmac4(acc[e], aux[e], xb[((1 + e) * R + r) * V], x);
            }
            __syncthreads();
            if (tid < 32) issue(j + ST);
        }
        if (f0 == 0) {
#pragma unroll
            for (int e = 0; e < E; ++e) {  // packed bin 0: (H_0 X_0, H_N X_N) as two real products
                acc[e].x += aux[e];
                acc[e].y = aux[e];
            }
        }
        if (G == 1) {
#pragma unroll
            for (int e = 0; e < E; ++e) reinterpret_cast<float4*>(s_yb + (size_t)e * N)[f0] = acc[e];
        } else {
#pragma unroll
            for (int e = 0; e < E; ++e) s_red[((size_t)g * V + f0) * E + e] = acc[e];
            __syncthreads();
            for (int i = tid; i < V * E; i += NT) {
                const int f = i / E, e = i % E;
                float4 sum = s_red[(size_t)f * E + e];
                for (int gg = 1; gg < G; ++gg) sum = f4add(sum, s_red[((size_t)gg * V + f) * E + e]);
                reinterpret_cast<float4*>(s_yb + (size_t)e * N)[f] = sum;
            }
        }
        __syncthreads();

        // ---- K5: inverse real FFT, hop-2 overlap-add.
        for (int e = 0; e < E; ++e) {
            for (int i = tid; i < N; i += NT) s_fb[i] = tangle_packed(s_yb + (size_t)e * N, N, i, s_pk);
            __syncthreads();
            const float* yf = reinterpret_cast<const float*>(fft_stockham<true, NC>(s_fb, s_fa, N, s_tw, false, tid, NT));
            const float sc = 1.0f / (float)N;
            float* A = p.ola + ((long)s * E + e) * 3 * L;
            float* o = p.out + ((long)s * E + e) * p.out_stride;
            for (int u = tid; u < L; u += NT) {
                const float y0 = yf[u] * sc, y1 = yf[L + u] * sc, y2 = yf[2 * L + u] * sc, y3 = yf[3 * L + u] * sc;
                o[u] = 0.5f * (y0 + A[u]);
                A[u] = y1 + A[L + u];
                A[L + u] = y2 + A[2 * L + u];
                A[2 * L + u] = y3;
            }
            __syncthreads();
        }
    }
}

// ============================================================================
// Hop-blocked kernel: the same per-hop semantics, processed J = 2*JH hops at a
// time when a call carries several hops (tvolap_process_hops). Within a block
// all J forward FFTs run first (spread over the cluster), then the MAC for the
// J outputs reuses every loaded spectrum: output i of parity group g (hop
// l0+g+2i) needs X_{l0+g+2(i-m)}, so a sliding register window over the
// delay line serves all JH outputs of a group with ONE delay-line load per
// partition, and a filter slice shared by those hops is loaded once instead of
// JH times. Every output is still the same sum over m in the same order, so
// results equal hop-by-hop processing. Ring depth D >= M + JH keeps the slots a
// block writes ahead from colliding with slots its earlier hops still read.
// ============================================================================
// Staging depth of the unified MAC: m-steps whose delay-line / filter float4s are in flight
// (cp.async, L2 -> shared) per thread ahead of the FMAs.
constexpr int kMacStages = 4;

// MAC work mapping of the hop-blocked kernel: per thread one float4 (two packed bins) for both
// parity groups (set engines, J <= 8), one float2 (one bin) for both parity groups (set engines,
// J = 16: half the accumulator registers per output), or one float4 of one parity group (bank).
enum MacMap { kUni4, kUni2, kParity };
__host__ __device__ constexpr MacMap mac_map(bool bank, int J) { return bank ? kParity : (J <= 8 ? kUni4 : kUni2); }

struct BlockLayout {
    size_t tw, pk, win, xin, yb, fa, fb, red, stg, ola, tdr, total;
    // fa | fb (FFT ping-pong) are idle during the MAC: the unified MAC's per-thread staging ring
    // and the partition-group partial sums (red) alias them; red is written only after every
    // thread has drained its ring, and is consumed before the inverse FFT reuses fa.
    __host__ __device__ BlockLayout(int L, int P, int E, int J, bool bank, int threads) {
        const size_t N = 2 * (size_t)L;
        const size_t fpc = (J + P - 1) / P;  // frames owned per CTA
        const size_t Np = N / P;
        tw = 0;
        pk = align16(tw + N * sizeof(float2));
        win = align16(pk + (N + 2) * sizeof(float2));
        xin = align16(win + N * sizeof(float));
        yb = align16(xin + (size_t)(J + 1) * L * sizeof(float));  // [history | J hops]
        fa = align16(yb + (size_t)J * E * Np * sizeof(float2));
        fb = align16(fa + fpc * E * N * sizeof(float2));
        const size_t V = Np / 2;
        const MacMap mm = mac_map(bank, J);
        const size_t W = mm == kUni4 ? V : 2 * V;  // work items per partition group
        const size_t qmax = W < (size_t)threads ? threads / W : 1;
        const size_t red_bytes = qmax > 1 ? qmax * J * E * V * sizeof(float4) : 0;
        red = fa;
        stg = fa;
        const size_t stg_bytes = mm == kUni4 ? (size_t)threads * kMacStages * (2 + E) * sizeof(float4) : 0;
        size_t end = fb + fpc * E * N * sizeof(float2);
        if (red + red_bytes > end) end = red + red_bytes;
        if (stg + stg_bytes > end) end = stg + stg_bytes;
        ola = align16(end);
        // time-domain receive buffer: the 4 quarter-slices of every frame of the block at this
        // CTA's output samples, pushed by the frame owners over DSMEM [J][E][4][L/P]
        tdr = align16(ola + (size_t)E * 3 * (L / P) * sizeof(float));
        total = align16(tdr + (size_t)J * E * 4 * (L / P) * sizeof(float));
    }
};

__device__ __forceinline__ void cluster_arrive(int P) {
    if (P > 1) asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void cluster_wait(int P) {
    if (P > 1) asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

__device__ __forceinline__ void block_sync(int P) {
    if (P > 1)
        cg::this_cluster().sync();
    else
        __syncthreads();
}

// BANK = false: filter-set engines (one set for every hop of a block) — only the unified
// mapping (JH <= 4) or the per-parity shared mapping (JH == 8) is compiled. BANK = true:
// per-hop bank selections — per-parity mapping with shared or per-output filter loads.
template <int E, int JH, bool BANK, int NC, bool SW = false>
__global__ void __launch_bounds__(256, 2) tvolap_block_kernel(const HopParams p, const int Q) {
    constexpr int J = 2 * JH;
    extern __shared__ __align__(16) unsigned char smem[];
    const int L = NC ? NC / 2 : p.L, N = 2 * L, M = p.M, D = p.D, P = p.P;
    const int tid = threadIdx.x, NT = blockDim.x;
    const int s = blockIdx.x / P;
    const int r = blockIdx.x % P;
    const BlockLayout lay(L, P, E, J, BANK, NT);
    (void)Q;
    PHASE_START();
    TL_BEGIN(0);
    float2* s_tw = reinterpret_cast<float2*>(smem + lay.tw);
    float2* s_pk = reinterpret_cast<float2*>(smem + lay.pk);
    float* s_win = reinterpret_cast<float*>(smem + lay.win);
    float* s_xin = reinterpret_cast<float*>(smem + lay.xin);
    float2* s_fa = reinterpret_cast<float2*>(smem + lay.fa);
    float2* s_fb = reinterpret_cast<float2*>(smem + lay.fb);
    float2* s_yb = reinterpret_cast<float2*>(smem + lay.yb);
    float4* s_red = reinterpret_cast<float4*>(smem + lay.red);
    float* s_ola = reinterpret_cast<float*>(smem + lay.ola);

    const int Np = N / P, V = Np / 2, Lp = L / P;
    // all of L, N, P, Np, V, Lp are powers of two: index math by shifts (no runtime divisions)
    const int lgL = 31 - __clz(L), lgN = lgL + 1, lgP = 31 - __clz(P);
    const int lgNp = lgN - lgP, lgV = lgNp - 1, lgLp = lgL - lgP, lgN2 = lgN - 1;
    const long spec4 = N / 2;
    const int W = 2 * V;             // (parity group, float4) work items
    const int q = tid / W;           // partition group (Q groups when W < NT)
    const int m0 = (int)((long)q * M / Q), m1 = (int)((long)(q + 1) * M / Q);

    for (int i = tid; i < N; i += NT) {
        s_tw[i] = p.tw[i];
        s_win[i] = p.win[i];
    }
    for (int i = tid; i <= N; i += NT) s_pk[i] = p.pk[i];
    // programmatic dependent launch: everything above reads constant tables only; from here on
    // the previous grid's state (history, OLA, delay line, pool, inputs) must be complete
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    float* xcur = s_xin;  // this block's inputs: [history | J hops]
    for (int i = tid; i < L; i += NT) xcur[i] = p.hist[(long)s * L + i];
    // hops b .. b+J-1 of this source into xcur[L..] (cp.async; lands while the block's MAC runs)
    const bool in_vec = (L & 3) == 0 && (p.in_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(p.in) & 15) == 0;
    // Switching mode (tvolap_process_switching): blocks end at switch boundaries; the next
    // switch's partitions are transformed by this launch inside the cluster-barrier gaps.
    // (a separate instantiation, SW = true, so the plain launches carry none of this code)
    const bool swm = SW && p.sw_count > 0;
    auto block_len = [&](int b) {
        int jn = min(J, p.n_hops - b);
        if (swm) jn = min(jn, (b / p.sw_period + 1) * p.sw_period - b);
        return jn;
    };
    auto prefetch_block = [&](int b) {
        const int jn = block_len(b);
        const float* src = p.in + (long)s * p.in_stride + (long)b * L;
        if (in_vec) {
            for (int i = 4 * tid; i < jn * L; i += 4 * NT) cp_async16(xcur + L + i, src + i);
        } else {
            for (int i = tid; i < jn * L; i += NT) {
                const unsigned sa = (unsigned)__cvta_generic_to_shared(xcur + L + i);
                asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(src + i));
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    prefetch_block(0);
    if (p.new_ir) {  // latch a staged filter set: transform it here (K4) while block 0's input lands
        __syncthreads();
        fused_partition<NC>(p, s, r, P, s_fa, s_fb, ((J + P - 1) / P) * E, lay.ola - lay.fa, s_tw, s_pk, tid,
                            NT);
        block_sync(P);
    }
    // K4 work units of this CTA for a switch: partitions m = r + u P, one warp per unit with a
    // warp-private buffer in the fa | fb | red area (idle in the barrier gaps it runs in).
    const int warp = tid >> 5, lane = tid & 31;
    const int k4_slots = max(1, min(NT >> 5, (int)((lay.ola - lay.fa) / (N * sizeof(float2)))));
    // one unit per warp per gap (same-box A/B: two lockstep units per warp in the first gap
    // measured 2.45 vs 2.37 us/hop on C2 — the longer second gap absorbs half the work better)
    const int k4_per_gap = k4_slots;
    const int k4_units = r < M ? (M - r + P - 1) / P : 0;
    auto k4_range = [&](const float* ir, int entry, int u0, int u1) {
        if constexpr (SW && NC != 0 && NC <= 1024 && !BANK) {
            const float* h = ir + (long)s * p.sw_ir_stride;
            const bool vec = (p.sw_ir_stride & 1) == 0 && (reinterpret_cast<uintptr_t>(ir) & 7) == 0;
            auto load_unit = [&](int u, int n) -> float2 {
                const long i0 = (long)(r + u * P) * NC + 2 * n;
                if (vec && i0 + 1 < p.sw_ir_len) return __ldcs(reinterpret_cast<const float2*>(h + i0));
                return make_float2(i0 < p.sw_ir_len ? h[i0] : 0.f, i0 + 1 < p.sw_ir_len ? h[i0 + 1] : 0.f);
            };
            auto store_unit = [&](const float2* buf, int u) {
                untangle_pairs_warp(buf, NC, s_pk, p.pool_w + ((long)(entry + s) * M + r + u * P) * NC, lane);
            };
            if (warp >= k4_slots) return;
            float2* buf = s_fa + (size_t)warp * NC;
            for (int u = u0 + warp; u < u1; u += k4_slots) {
                fft_warp4<false, NC, true>(buf, p.tw + NC, lane, [&](int, int n) { return load_unit(u, n); });
                store_unit(buf, u);
                __syncwarp();
            }
        } else {
            (void)ir, (void)entry, (void)u0, (void)u1;
        }
    };
    int cur_entry = p.entry_base;  // pool entry (of source 0) of the running filter set
    if (SW && swm && p.sw_entry[0] >= 0) {  // switch 0 at the first hop: transform it before any MAC
        __syncthreads();
        k4_range(p.sw_irs[0], p.sw_entry[0], 0, k4_units);
        cur_entry = p.sw_entry[0];
        block_sync(P);
    }
    const float* k4_ir = nullptr;  // the next switch's set, transformed during this period
    int k4_entry = -1, k4_done = 0;
    for (int i = tid; i < E * 3 * Lp; i += NT) {
        const int e = i / (3 * Lp), rem = i % (3 * Lp), j = rem / Lp, u = rem % Lp;
        s_ola[i] = p.ola[((long)s * E + e) * 3 * L + j * L + r * Lp + u];
    }

    const float4* ring4 = reinterpret_cast<const float4*>(p.ring);
    const float4* pool4 = reinterpret_cast<const float4*>(p.pool);
    cg::cluster_group cluster = cg::this_cluster();
    PHASE_MARK(11);

    for (int b0 = 0, jb = 0; b0 < p.n_hops; b0 += jb) {
        const long l0 = p.hop0 + b0;
        jb = block_len(b0);
        bool period_end = false;
        if (SW && swm) {
            const int k = b0 / p.sw_period;
            if (b0 % p.sw_period == 0) {  // a new period: latch switch k, prepare switch k + 1
                if (k > 0 && p.sw_entry[k] >= 0) cur_entry = p.sw_entry[k];
                k4_ir = nullptr;
                if (k + 1 < p.sw_count && p.sw_entry[k + 1] >= 0) {
                    k4_ir = p.sw_irs[k + 1];
                    k4_entry = p.sw_entry[k + 1];
                }
                k4_done = 0;
            }
            period_end = (b0 + jb) % p.sw_period == 0 || b0 + jb >= p.n_hops;
        }
        if (b0 + jb >= p.n_hops) asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
        // delay-line slots: hop l0 + k lives in slot ((l0 + k) >> 1) mod D of parity (l0 + k) & 1;
        // one 64-bit modulo per block, then small int offsets with a single wrap
        const int sl0 = (int)((l0 >> 1) % D), odd0 = (int)(l0 & 1);
        auto slot_of = [&](int k) {
            const int sl = sl0 + ((odd0 + k) >> 1);
            return sl >= D ? sl - D : sl;
        };
        auto wrapD = [&](int x) { return x < 0 ? x + D : (x >= D ? x - D : x); };
        // ---- inputs: this block's landed (prefetched during the previous block)
        asm volatile("cp.async.wait_all;\n" ::: "memory");
        __syncthreads();
        PHASE_MARK(0);

        // ---- K1/K2: this CTA's frames (j = r, r+P, ...): window, FFT, whole spectrum into the ring.
        const int nf = jb > r ? (jb - r + P - 1) / P : 0;
        for (int i = tid; i < nf * L; i += NT) {
            const int f = i >> lgL, jj = i & (L - 1);
            const float* xs = xcur + (size_t)(r + f * P) * L;  // (previous hop | this hop)
            s_fa[(size_t)f * N + jj] = make_float2(xs[2 * jj] * s_win[2 * jj], xs[2 * jj + 1] * s_win[2 * jj + 1]);
        }
        __syncthreads();
        // history for the next block = last input hop of this block; then start the next
        // block's input copy into the (now free) hop area
        for (int i = tid; i < L; i += NT) xcur[i] = xcur[(size_t)jb * L + i];
        __syncthreads();
        if (b0 + jb < p.n_hops) prefetch_block(b0 + jb);
        if (nf > 0) {
            const float2* Z = fft_batch<false, NC>(s_fa, s_fb, N, nf, s_tw, true, tid, NT);
            for (int f = 0; f < nf; ++f) {
                const int k = r + f * P;
                float2* ringw = p.ring + (((long)s * 2 + ((odd0 + k) & 1)) * D + slot_of(k)) * N;
                untangle_store<NC>(Z + (size_t)f * N, N, s_pk, ringw, tid, NT);
            }
        }
        PHASE_MARK(1);
        if (SW && k4_ir) {  // ring writes visible cluster-wide; next switch's K4 units in the barrier gap
            __syncthreads();
            cluster_arrive(P);
            const int u1 = min(k4_units, k4_done + k4_per_gap);
            k4_range(k4_ir, k4_entry, k4_done, u1);
            k4_done = u1;
            __syncthreads();
            cluster_wait(P);
        } else {
            block_sync(P);  // ring writes of all frames visible cluster-wide
        }
        PHASE_MARK(2);

        // ---- K3: hop-blocked MAC over this CTA's bin slice.
        // Does every hop of the block use the same filter set (set engines: always)?
        bool all_same = true;
        int ent0 = cur_entry + s;
        if (p.sched) {
            ent0 = p.sched[(long)b0 * p.sched_stride + s];
            for (int jj = 1; jj < jb; ++jj) all_same &= p.sched[(long)(b0 + jj) * p.sched_stride + s] == ent0;
        }
        int Qeff;
        constexpr MacMap kMap = mac_map(BANK, J);
        if constexpr (kMap == kUni4) {
            // Unified mapping: one thread per float4 covers both parity groups, so each filter
            // slice is loaded once per block for all J outputs; two sliding delay-line windows.
            Qeff = V < NT ? NT / V : 1;
            const int qq = V < NT ? tid / V : 0;
            const int mu0 = (int)((long)qq * M / Qeff), mu1 = (int)((long)(qq + 1) * M / Qeff);
            constexpr int JU = JH <= 4 ? JH : 1;
            for (int f = (V >= NT ? tid : tid % V); f < V; f += (V >= NT ? NT : V)) {
                const float4* xr[2];
                int sbp[2];
#pragma unroll
                for (int g = 0; g < 2; ++g) {
                    xr[g] = ring4 + (((long)s * 2 + ((odd0 + g) & 1)) * D) * spec4 + (long)r * V + f;
                    sbp[g] = slot_of(g);
                }
                auto xs = [&](int g, int t) -> const float4* {  // window init only
                    return xr[g] + (long)wrapD(sbp[g] + t) * spec4;
                };
                // slot cursors for the next delay-line load (t = -m-1), decremented per partition
                int cur[2];
#pragma unroll
                for (int g = 0; g < 2; ++g) cur[g] = wrapD(sbp[g] - mu0 - 1);
                const float4* hb4[E];
#pragma unroll
                for (int e = 0; e < E; ++e) hb4[e] = pool4 + (((long)ent0 * E + e) * M) * spec4 + (long)r * V + f;
                float4 acc[2][JU][E];
                float aux[2][JU][E];
                float4 win[2][JU];
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int i = 0; i < JU; ++i) {
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            acc[g][i][e] = make_float4(0.f, 0.f, 0.f, 0.f);
                            aux[g][i][e] = 0.f;
                        }
                        win[g][i] = __ldcg(xs(g, i - mu0));
                    }
                // Per-thread staging ring in shared memory: step m's two delay-line float4s and
                // E filter float4s land in slot (m - mu0) % kMacStages via cp.async (L2 -> smem),
                // kMacStages steps ahead of the FMAs. Each thread reads back only what it copied
                // itself, so wait_group is the only synchronisation needed.
                float4* stg = reinterpret_cast<float4*>(smem + lay.stg) + tid;
                constexpr int CS = 2 + E;
                auto stage = [&](int mm, int k) {
                    if (mm < mu1) {
#pragma unroll
                        for (int g = 0; g < 2; ++g) {
                            cp_async16(stg + (size_t)(k * CS + g) * NT, xr[g] + (long)cur[g] * spec4);
                            cur[g] = cur[g] == 0 ? D - 1 : cur[g] - 1;
                        }
#pragma unroll
                        for (int e = 0; e < E; ++e)
                            cp_async16(stg + (size_t)(k * CS + 2 + e) * NT, hb4[e] + (long)mm * spec4);
                    }
                    asm volatile("cp.async.commit_group;\n" ::);
                };
                auto step = [&](int mm, int k) {
                    asm volatile("cp.async.wait_group %0;\n" ::"n"(kMacStages - 1));
                    float4 xn[2], hh[E];
#pragma unroll
                    for (int g = 0; g < 2; ++g) xn[g] = stg[(size_t)(k * CS + g) * NT];
#pragma unroll
                    for (int e = 0; e < E; ++e) hh[e] = stg[(size_t)(k * CS + 2 + e) * NT];
#pragma unroll
                    for (int g = 0; g < 2; ++g) {
#pragma unroll
                        for (int i = 0; i < JU; ++i)
#pragma unroll
                            for (int e = 0; e < E; ++e) cmac4(acc[g][i][e], aux[g][i][e], hh[e], win[g][i]);
#pragma unroll
                        for (int i = JU - 1; i > 0; --i) win[g][i] = win[g][i - 1];
                        win[g][0] = xn[g];
                    }
                    stage(mm + kMacStages, k);
                };
#pragma unroll
                for (int k = 0; k < kMacStages; ++k) stage(mu0 + k, k);
                int m = mu0;
                for (; m + kMacStages <= mu1; m += kMacStages) {
#pragma unroll
                    for (int k = 0; k < kMacStages; ++k) step(m + k, k);
                }
                for (int k = 0; m < mu1; ++m, ++k) step(m, k);
                asm volatile("cp.async.wait_all;\n" ::);
                if (Qeff > 1) __syncthreads();  // s_red aliases the staging rings (one f per thread here)
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int i = 0; i < JU; ++i) {
                        const int jj = g + 2 * i;
                        if (jj >= jb) continue;
#pragma unroll
                        for (int e = 0; e < E; ++e) {
                            float4 a = acc[g][i][e];
                            if (r == 0 && f == 0) {  // packed bin 0: two real products
                                a.x += aux[g][i][e];
                                a.y = aux[g][i][e];
                            }
                            if (Qeff == 1)
                                reinterpret_cast<float4*>(s_yb + ((size_t)jj * E + e) * Np)[f] = a;
                            else
                                s_red[(((size_t)qq * J + jj) * E + e) * V + f] = a;
                        }
                    }
            }
        } else if constexpr (kMap == kUni2) {
            // Unified float2 mapping (16-hop blocks): one thread per packed bin covers both parity
            // groups, 8 outputs each, so every filter and delay-line element is loaded once per
            // 16 hops. Partition groups: Qeff = threads / Np (same count as the per-parity mapping).
            static_assert(E == 1, "filter-set engines have one ear");
            Qeff = Np < NT ? NT / Np : 1;
            const int qq = Np < NT ? tid / Np : 0;
            const int mu0 = (int)((long)qq * M / Qeff), mu1 = (int)((long)(qq + 1) * M / Qeff);
            const float2* ring2 = p.ring;
            const float2* pool2 = p.pool;
            for (int f = (Np >= NT ? tid : tid % Np); f < Np; f += (Np >= NT ? NT : Np)) {
                // the packed bin 0 (r == 0, f == 0) needs the Nyquist product: warps holding it
                // run the variant with the extra accumulator (warp-uniform branch)
                const bool pkw = __any_sync(0xffffffffu, r == 0 && f == 0);
                auto mac = [&](auto pk_tag) {
                    constexpr bool PK = decltype(pk_tag)::value;
                    const float2* xr[2];
                    int sbp[2];
                    int cur[2];
#pragma unroll
                    for (int g = 0; g < 2; ++g) {
                        xr[g] = ring2 + (((long)s * 2 + ((odd0 + g) & 1)) * D) * N + (long)r * Np + f;
                        sbp[g] = slot_of(g);
                        cur[g] = wrapD(sbp[g] - mu0 - 1);
                    }
                    const float2* hb = pool2 + ((long)ent0 * M) * N + (long)r * Np + f;
                    float2 acc[2][JH];
                    float aux[2][PK ? JH : 1];
                    float2 win[2][JH];
#pragma unroll
                    for (int g = 0; g < 2; ++g)
#pragma unroll
                        for (int i = 0; i < JH; ++i) {
                            acc[g][i] = make_float2(0.f, 0.f);
                            if constexpr (PK) aux[g][i] = 0.f;
                            win[g][i] = __ldcg(xr[g] + (long)wrapD(sbp[g] + i - mu0) * N);
                        }
                    auto mac_step = [&](const float2 (&xn)[2], const float2 h) {
#pragma unroll
                        for (int g = 0; g < 2; ++g) {
#pragma unroll
                            for (int i = 0; i < JH; ++i) {
                                float2& a = acc[g][i];
                                const float2 x = win[g][i];
                                a.x = fmaf(h.x, x.x, a.x);
                                a.x = fmaf(-h.y, x.y, a.x);
                                a.y = fmaf(h.x, x.y, a.y);
                                a.y = fmaf(h.y, x.x, a.y);
                                if constexpr (PK) aux[g][i] = fmaf(h.y, x.y, aux[g][i]);
                            }
#pragma unroll
                            for (int i = JH - 1; i > 0; --i) win[g][i] = win[g][i - 1];
                            win[g][0] = xn[g];
                        }
                    };
                    int m = mu0;
                    constexpr int U = 4;  // same-box A/B: U = 2 +1.5 %, one aux-everywhere variant +9 %
                    for (; m + U <= mu1; m += U) {
                        float2 xn[U][2], hh[U];
#pragma unroll
                        for (int u = 0; u < U; ++u) {
#pragma unroll
                            for (int g = 0; g < 2; ++g) {
                                xn[u][g] = __ldcg(xr[g] + (long)cur[g] * N);
                                cur[g] = cur[g] == 0 ? D - 1 : cur[g] - 1;
                            }
                            hh[u] = __ldcg(hb + (long)(m + u) * N);
                        }
#pragma unroll
                        for (int u = 0; u < U; ++u) mac_step(xn[u], hh[u]);
                    }
                    for (; m < mu1; ++m) {
                        float2 xn[2];
#pragma unroll
                        for (int g = 0; g < 2; ++g) {
                            xn[g] = __ldcg(xr[g] + (long)cur[g] * N);
                            cur[g] = cur[g] == 0 ? D - 1 : cur[g] - 1;
                        }
                        mac_step(xn, __ldcg(hb + (long)m * N));
                    }
                    float2* red2 = reinterpret_cast<float2*>(s_red);
#pragma unroll
                    for (int g = 0; g < 2; ++g)
#pragma unroll
                        for (int i = 0; i < JH; ++i) {
                            const int jj = g + 2 * i;
                            if (jj >= jb) continue;
                            float2 a = acc[g][i];
                            if constexpr (PK) {
                                if (r == 0 && f == 0) {  // packed bin 0: two real products
                                    a.x += aux[g][i];
                                    a.y = aux[g][i];
                                }
                            }
                            if (Qeff == 1)
                                s_yb[(size_t)jj * Np + f] = a;
                            else
                                red2[((size_t)qq * J + jj) * Np + f] = a;
                        }
                };
                if (pkw)
                    mac(std::true_type{});
                else
                    mac(std::false_type{});
            }
        } else {
        Qeff = W < NT ? NT / W : 1;
        // Per-parity mapping (W >= NT: threads stride over the work items; W < NT: Qeff groups of W).
        for (int w = (W >= NT ? tid : tid % W); w < W; w += (W >= NT ? NT : W)) {
            const int g = w / V, f = w - g * V;
            const int par = (odd0 + g) & 1;
            const int sb = slot_of(g);
            const int ni = jb > g ? (jb - g + 1) / 2 : 0;  // outputs of this parity group
            const float4* xr = ring4 + (((long)s * 2 + par) * D) * spec4 + (long)r * V + f;
            auto xslot = [&](int t) -> const float4* {  // window init only
                return xr + (long)wrapD(sb + t) * spec4;
            };
            int cur = wrapD(sb - m0 - 1);  // slot of the next load (t = -m-1)
            auto xnext = [&]() -> float4 {
                const float4 v = __ldcg(xr + (long)cur * spec4);
                cur = cur == 0 ? D - 1 : cur - 1;
                return v;
            };
            int ent[JH];
            bool shared = true;
#pragma unroll
            for (int i = 0; i < JH; ++i) {
                const int jj = g + 2 * i;
                ent[i] = p.sched ? p.sched[(long)(b0 + min(jj, jb - 1)) * p.sched_stride + s] : p.entry_base + s;
                if (i < ni && ent[i] != ent[0]) shared = false;
            }
            float4 acc[JH][E];
            float aux[JH][E];
            float4 win[JH];
#pragma unroll
            for (int i = 0; i < JH; ++i) {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    acc[i][e] = make_float4(0.f, 0.f, 0.f, 0.f);
                    aux[i][e] = 0.f;
                }
                win[i] = __ldcg(xslot(i - m0));  // X_{t}, t = i - m
            }
            if (!BANK || shared) {
                const float4* hb4[E];
#pragma unroll
                for (int e = 0; e < E; ++e) hb4[e] = pool4 + (((long)ent[0] * E + e) * M) * spec4 + (long)r * V + f;
                int m = m0;
                constexpr int U = JH >= 8 ? 2 : 4;
                for (; m + U <= m1; m += U) {
                    float4 xn[U], hh[U][E];
#pragma unroll
                    for (int u = 0; u < U; ++u) {
                        xn[u] = xnext();
#pragma unroll
                        for (int e = 0; e < E; ++e) hh[u][e] = __ldcg(hb4[e] + (long)(m + u) * spec4);
                    }
#pragma unroll
                    for (int u = 0; u < U; ++u) {
#pragma unroll
                        for (int i = 0; i < JH; ++i)
#pragma unroll
                            for (int e = 0; e < E; ++e) cmac4(acc[i][e], aux[i][e], hh[u][e], win[i]);
#pragma unroll
                        for (int i = JH - 1; i > 0; --i) win[i] = win[i - 1];
                        win[0] = xn[u];
                    }
                }
                for (; m < m1; ++m) {
                    const float4 xn = xnext();
#pragma unroll
                    for (int e = 0; e < E; ++e) {
                        const float4 h = __ldcg(hb4[e] + (long)m * spec4);
#pragma unroll
                        for (int i = 0; i < JH; ++i) cmac4(acc[i][e], aux[i][e], h, win[i]);
                    }
#pragma unroll
                    for (int i = JH - 1; i > 0; --i) win[i] = win[i - 1];
                    win[0] = xn;
                }
            } else {
                // per-output filters (bank switching inside the block). Two ears: 32-bit float4
                // offsets into the pool, one register each instead of a pointer pair (same-box:
                // C3 5.08e9 vs 4.78e9); one ear keeps pointers (C5 1.07e9 vs 0.94e9 with offsets)
                //
                // L2 bulk prefetch (cp.async.bulk.prefetch.L2, no registers): every per-output
                // filter row and delay-line row is requested kPfDist partitions ahead by one lane
                // per (output, ear) and one lane for the delay line, so the 16-byte loads below
                // find their lines in L2 instead of waiting on HBM; bytes in flight towards HBM no
                // longer depend on the register budget.
                const int ln = tid & 31;
                const int fw = f & ~31;  // this warp's float4 column range [fw, fw + 32) of the slice
                int pf_ent = -1, pf_e = 0;
#pragma unroll
                for (int i = 0; i < JH; ++i)
#pragma unroll
                    for (int e = 0; e < E; ++e)
                        if (ln == i * E + e && i < ni) pf_ent = ent[i], pf_e = e;
                const bool row_whole = V == 32 && P == 1;  // warp slice == whole row: rows contiguous
                auto prefetch_rows = [&](const float4* base, int rows) {  // rows consecutive rows from base
                    if (row_whole) {
                        l2_prefetch(base, (unsigned)rows * 512u);
                    } else {
                        for (int k = 0; k < rows; ++k) l2_prefetch(base + (long)k * spec4, 512u);
                    }
                };
                // (only where a warp covers 32 consecutive float4 columns of one parity group)
                const bool pf_on = (V & 31) == 0;
                auto prefetch_chunk = [&](int mc) {  // partitions [mc, mc + kPfRows) of this thread's group
                    const int me = min(mc + kPfRows, m1);
                    if (!pf_on || mc >= me) return;
                    if (pf_ent >= 0) {
                        prefetch_rows(pool4 + (((long)pf_ent * E + pf_e) * M + mc) * spec4 + (long)r * V + fw, me - mc);
                    } else if (ln == 31) {  // delay line: slots of t = -m-1 run downwards from sb - mc - 1
                        const int hi = wrapD(sb - mc - 1), lo = wrapD(sb - me);
                        const float4* xw = xr - f + fw;
                        if (lo <= hi) {
                            prefetch_rows(xw + (long)lo * spec4, hi - lo + 1);
                        } else {
                            prefetch_rows(xw, hi + 1);
                            prefetch_rows(xw + (long)lo * spec4, D - lo);
                        }
                    }
                };
#ifndef TVOLAP_NO_L2PF
                prefetch_chunk(m0 + kPfRows);
#endif
                if constexpr (E == 2) {
                    unsigned hoff[JH][E];
#pragma unroll
                    for (int i = 0; i < JH; ++i)
#pragma unroll
                        for (int e = 0; e < E; ++e)
                            hoff[i][e] = (unsigned)((((long)ent[i] * E + e) * M) * spec4 + (long)r * V + f);
                    for (int mc = m0; mc < m1; mc += kPfRows) {
#ifndef TVOLAP_NO_L2PF
                        prefetch_chunk(mc + kPfDist);
#endif
                        const int me = min(mc + kPfRows, m1);
                        unsigned mo = (unsigned)((long)mc * spec4);
#pragma unroll 2
                        for (int m = mc; m < me; ++m, mo += (unsigned)spec4) {
                            const float4 xn = xnext();
#pragma unroll
                            for (int i = 0; i < JH; ++i)
#pragma unroll
                                for (int e = 0; e < E; ++e)
                                    cmac4(acc[i][e], aux[i][e], __ldcg(pool4 + (hoff[i][e] + mo)), win[i]);
#pragma unroll
                            for (int i = JH - 1; i > 0; --i) win[i] = win[i - 1];
                            win[0] = xn;
                        }
                    }
                } else {
                    const float4* hbi[JH][E];
#pragma unroll
                    for (int i = 0; i < JH; ++i)
#pragma unroll
                        for (int e = 0; e < E; ++e) hbi[i][e] = pool4 + (((long)ent[i] * E + e) * M) * spec4 + (long)r * V + f;
                    for (int mc = m0; mc < m1; mc += kPfRows) {
#ifndef TVOLAP_NO_L2PF
                        prefetch_chunk(mc + kPfDist);
#endif
                        const int me = min(mc + kPfRows, m1);
#pragma unroll 2
                        for (int m = mc; m < me; ++m) {
                            const float4 xn = xnext();
#pragma unroll
                            for (int i = 0; i < JH; ++i)
#pragma unroll
                                for (int e = 0; e < E; ++e) cmac4(acc[i][e], aux[i][e], __ldcg(hbi[i][e] + (long)m * spec4), win[i]);
#pragma unroll
                            for (int i = JH - 1; i > 0; --i) win[i] = win[i - 1];
                            win[0] = xn;
                        }
                    }
                }
            }
#pragma unroll
            for (int i = 0; i < JH; ++i) {
                const int jj = g + 2 * i;
                if (i >= ni) continue;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    float4 a = acc[i][e];
                    if (r == 0 && f == 0) {  // packed bin 0: two real products
                        a.x += aux[i][e];
                        a.y = aux[i][e];
                    }
                    if (Qeff == 1)
                        reinterpret_cast<float4*>(s_yb + ((size_t)jj * E + e) * Np)[f] = a;
                    else
                        s_red[(((size_t)q * J + jj) * E + e) * V + f] = a;
                }
            }
        }
        }
        PHASE_MARK(3);
        if (Qeff > 1) {
            __syncthreads();
            for (int i = tid; i < jb * E * V; i += NT) {
                const int f = i & (V - 1), je = i >> lgV;  // je = jj * E + e
                float4 sum = s_red[(size_t)je * V + f];
                for (int qq = 1; qq < Qeff; ++qq) sum = f4add(sum, s_red[((size_t)qq * J * E + je) * V + f]);
                reinterpret_cast<float4*>(s_yb + (size_t)je * Np)[f] = sum;
            }
        }
        PHASE_MARK(4);
        if (SW && k4_ir) {  // Y slices published; more K4 units (all that remain at the period's end)
            __syncthreads();
            cluster_arrive(P);
            const int u1 = period_end ? k4_units : min(k4_units, k4_done + k4_per_gap);
            k4_range(k4_ir, k4_entry, k4_done, u1);
            k4_done = u1;
            __syncthreads();
            cluster_wait(P);
        } else {
            block_sync(P);  // Y slices of all frames published
        }
        PHASE_MARK(5);

        // ---- K5a: this CTA's frames: gather Y over DSMEM, tangle, inverse FFT.
        const int nt = nf * E;  // transforms
        for (int i = tid; i < nt * (N / 2); i += NT) {  // float4 granularity gather
            const int t = i >> lgN2, k4 = i & (N / 2 - 1);
            const int f = t / E, e = t - f * E;
            const int jj = r + f * P;
            const int qsrc = k4 >> lgV;
            const float4* src = reinterpret_cast<const float4*>(s_yb + ((size_t)jj * E + e) * Np);
            if (qsrc != r) src = cluster.map_shared_rank(src, qsrc);
            reinterpret_cast<float4*>(s_fa + (size_t)t * N)[k4] = src[k4 - qsrc * (Np / 2)];
        }
        __syncthreads();
        for (int i = tid; i < nt * N; i += NT) {
            const int t = i >> lgN, kk = i & (N - 1);
            s_fb[(size_t)t * N + kk] = tangle_packed(s_fa + (size_t)t * N, N, kk, s_pk);
        }
        __syncthreads();
        if (nt > 0) fft_batch<true, NC>(s_fb, s_fa, N, nt, s_tw, false, tid, NT);
        // the result buffer depends only on the stage count (same in every CTA of the cluster)
        const int stages = fft_stage_count(N);
        const float* ytd = reinterpret_cast<const float*>((stages & 1) ? s_fa : s_fb);
        // time-domain frame (f, e) of this CTA = ytd[(f * E + e) * 2N ...] (unscaled); push each
        // frame's quarter-slices, scaled, to the CTAs that emit those output samples (DSMEM
        // stores: the OLA then reads only local shared memory, and no barrier has to protect
        // ytd from remote readers)
        float* s_tdr = reinterpret_cast<float*>(smem + lay.tdr);
        {
            const float sc = 1.0f / (float)N;
            if ((Lp & 3) == 0) {
                const int L4 = L >> 2, lgL4 = lgL - 2;
                for (int i = tid; i < nt * 4 * L4; i += NT) {  // (transform t, quarter d, float4 v)
                    const int v = i & (L4 - 1), td = i >> lgL4, d = td & 3, t = td >> 2;
                    const int f = t / E, e = t - f * E;
                    float4 y4 = reinterpret_cast<const float4*>(ytd + (size_t)t * 2 * N + (size_t)d * L)[v];
                    y4 = make_float4(y4.x * sc, y4.y * sc, y4.z * sc, y4.w * sc);
                    const int smp = 4 * v, q = smp >> lgLp, u = smp & (Lp - 1);
                    const int jj = r + f * P;
                    float* dst = s_tdr + ((size_t)(jj * E + e) * 4 + d) * Lp + u;
                    if (q != r) dst = cluster.map_shared_rank(dst, q);
                    *reinterpret_cast<float4*>(dst) = y4;
                }
            } else {
                for (int i = tid; i < nt * 4 * L; i += NT) {
                    const int smp = i & (L - 1), td = i >> lgL, d = td & 3, t = td >> 2;
                    const int f = t / E, e = t - f * E;
                    const float y = ytd[(size_t)t * 2 * N + (size_t)d * L + smp] * sc;
                    const int q = smp >> lgLp, u = smp & (Lp - 1);
                    const int jj = r + f * P;
                    float* dst = s_tdr + ((size_t)(jj * E + e) * 4 + d) * Lp + u;
                    if (q != r) dst = cluster.map_shared_rank(dst, q);
                    *dst = y;
                }
            }
        }
        PHASE_MARK(6);
        block_sync(P);  // all frames' time-domain slices delivered
        PHASE_MARK(7);

        // ---- K5b: hop-2 overlap-add for this CTA's sample slice, all frames of the block
        // (from the local receive buffer).
        for (int i = tid; i < E * Lp; i += NT) {
            const int e = i >> lgLp, u = i & (Lp - 1);
            const int ug = r * Lp + u;
            float* A = s_ola + e * 3 * Lp;
            float a0 = A[u], a1 = A[Lp + u], a2 = A[2 * Lp + u];
            float* o = p.out + ((long)s * E + e) * p.out_stride + (long)b0 * L + ug;
            constexpr int JC = J < 8 ? J : 8;  // frames gathered per chunk (register bound)
#pragma unroll
            for (int j0 = 0; j0 < J; j0 += JC) {
                if (j0 >= jb) break;
                float y[JC][4];
#pragma unroll
                for (int jc = 0; jc < JC; ++jc) {
                    const int jj = j0 + jc;
                    if (jj < jb) {
                        const float* yf = s_tdr + (size_t)(jj * E + e) * 4 * Lp + u;
#pragma unroll
                        for (int d = 0; d < 4; ++d) y[jc][d] = yf[d * Lp];
                    } else {
#pragma unroll
                        for (int d = 0; d < 4; ++d) y[jc][d] = 0.f;
                    }
                }
#pragma unroll
                for (int jc = 0; jc < JC; ++jc) {
                    const int jj = j0 + jc;
                    if (jj >= jb) break;
                    // pending = contributions of earlier frames: rolling (a0, a1, a2)
                    o[(long)jj * L] = 0.5f * (y[jc][0] + a0);
                    a0 = a1 + y[jc][1];
                    a1 = a2 + y[jc][2];
                    a2 = y[jc][3];
                }
            }
            A[u] = a0;
            A[Lp + u] = a1;
            A[2 * Lp + u] = a2;
        }
        PHASE_MARK(8);
        PHASE_MARK(9);
        // No cluster barrier here: peers read nothing of this CTA after the time-domain barrier
        // (its Y slices are protected by the next block's first barrier, which peers reach only
        // after their gather), and the next block's pushes into s_tdr come after its Y barrier,
        // which this CTA reaches only after the overlap-add above. (Intra-CTA, the next block
        // starts with __syncthreads; the write-back below has its own.)
        PHASE_MARK(10);
#ifdef TVOLAP_PHASE_PROF
        if (tid == 0) atomicAdd(&g_phase[12], 1ull);
#endif
    }
    __syncthreads();  // the OLA threads' last s_ola updates before the state write-back
    asm volatile("cp.async.wait_all;\n" ::);
    if (r == 0)
        for (int i = tid; i < L; i += NT) p.hist[(long)s * L + i] = xcur[i];
    for (int i = tid; i < E * 3 * Lp; i += NT) {
        const int e = i / (3 * Lp), rem = i % (3 * Lp), j = rem / Lp, u = rem % Lp;
        p.ola[((long)s * E + e) * 3 * L + j * L + r * Lp + u] = s_ola[i];
    }
    TL_END(0);
}

// K4: transform IR slices into packed partition spectra (partition.cpp:20-51).
template <int NC>
__global__ void __launch_bounds__(256) partition_kernel(int L, int M, long rows, const float* __restrict__ ir,
                                                        long ir_stride, long ir_len, float2* __restrict__ pool,
                                                        long row0, const float2* __restrict__ tw,
                                                        const float2* __restrict__ pk, int nf) {
    if constexpr (NC != 0) L = NC / 2;
    const bool vec = L >= 2 && (ir_stride & 3) == 0 && (reinterpret_cast<uintptr_t>(ir) & 15) == 0;
    // nf partitions per CTA iteration through one batched FFT (fewer barriers per transform)
    extern __shared__ __align__(16) unsigned char smem[];
    const int N = 2 * L, tid = threadIdx.x, NT = blockDim.x;
    float2* s_tw = reinterpret_cast<float2*>(smem);
    float2* s_pk = s_tw + N;
    float2* s_fa = s_pk + N + 2;
    float2* s_fb = s_fa + (size_t)nf * N;
    for (int i = tid; i < N; i += NT) s_tw[i] = tw[i];
    for (int i = tid; i <= N; i += NT) s_pk[i] = pk[i];
    __syncthreads();
    const long tasks = rows * M;
    const int lgL = 31 - __clz(L);  // L a power of two: shifts, no divisions
    for (long t0 = (long)blockIdx.x * nf; t0 < tasks; t0 += (long)gridDim.x * nf) {
        const int nt = (int)min((long)nf, tasks - t0);
        const long row0t = t0 / M;  // one 64-bit division per group
        const int m0t = (int)(t0 - row0t * M);
        if (vec) {  // 16-byte loads: z[j], z[j+1] = (h[2j], h[2j+1]), (h[2j+2], h[2j+3])
            const int L2 = L >> 1, lgL2 = lgL - 1;
            for (int i = tid; i < nt * L2; i += NT) {
                const int f = i >> lgL2, j = (i & (L2 - 1)) * 2;
                int m = m0t + f;
                long row = row0t;
                while (m >= M) m -= M, ++row;
                const long i0 = (long)m * N + 2 * j;
                const float* h = ir + row * ir_stride;
                float4 v;
                if (i0 + 3 < ir_len) {
                    v = __ldcs(reinterpret_cast<const float4*>(h + i0));
                } else {
                    v.x = i0 < ir_len ? h[i0] : 0.f;
                    v.y = i0 + 1 < ir_len ? h[i0 + 1] : 0.f;
                    v.z = i0 + 2 < ir_len ? h[i0 + 2] : 0.f;
                    v.w = i0 + 3 < ir_len ? h[i0 + 3] : 0.f;
                }
                reinterpret_cast<float4*>(s_fa + (size_t)f * N)[j >> 1] = v;
            }
        } else {
            for (int i = tid; i < nt * L; i += NT) {
                const int f = i >> lgL, j = i & (L - 1);
                int m = m0t + f;
                long row = row0t;
                while (m >= M) m -= M, ++row;
                const long i0 = (long)m * N + 2 * j;
                const float* h = ir + row * ir_stride;
                const float a = i0 < ir_len ? h[i0] : 0.f;
                const float b = i0 + 1 < ir_len ? h[i0 + 1] : 0.f;
                s_fa[(size_t)f * N + j] = make_float2(a, b);
            }
        }
        __syncthreads();
        const float2* Z = fft_batch<false, NC>(s_fa, s_fb, N, nt, s_tw, true, tid, NT);
        for (int f = 0; f < nt; ++f)
            untangle_store<NC>(Z + (size_t)f * N, N, s_pk, pool + (row0 * M + t0 + f) * N, tid, NT);
        __syncthreads();
    }
}

// K4, one warp per partition (N <= 1024): no CTA barriers, a warp-private 8N-byte buffer, IR
// slices read straight into the first FFT stage's registers. Bit-identical to partition_kernel.
template <int NC>
// (same-box A/B for N = 1024: one CTA per SM without spills 248 us per C4 switch vs 225 us here)
__global__ void __launch_bounds__(256, 2) partition_warp_kernel(int M, long rows, const float* __restrict__ ir,
                                                             long ir_stride, long ir_len, float2* __restrict__ pool,
                                                             long row0, const float2* __restrict__ tw,
                                                             const float2* __restrict__ pk, int k4_prefetch) {
    constexpr int N = NC;
    extern __shared__ __align__(16) unsigned char smem[];
    float2* s_tw = reinterpret_cast<float2*>(smem);
    float2* s_pk = s_tw + N;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    float2* buf = reinterpret_cast<float2*>(smem + align16((2 * N + 2) * sizeof(float2))) + (size_t)warp * N;
    TL_BEGIN(1);
    (void)s_tw;  // the four-step tables are read through L1 (tw + N)
    // In-stream K4 under programmatic dependent launch: let the next hop launch get scheduled
    // now, and (below) finish only after the previous hop launch has completed, so the hop
    // launch that waits on this grid transitively waits on its predecessor too.
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
    for (int i = tid; i <= N; i += blockDim.x) s_pk[i] = pk[i];
    __syncthreads();
    const bool vec = (ir_stride & 1) == 0 && (reinterpret_cast<uintptr_t>(ir) & 7) == 0;
    const long tasks = rows * M;
    for (long t = (long)blockIdx.x * nw + warp; t < tasks; t += (long)gridDim.x * nw) {
        const long row = t / M;
        const int m = (int)(t - row * M);
        const float* h = ir + row * ir_stride;
        const long base = (long)m * N;  // partition m = IR samples [m N, (m + 1) N), N = 2L
        if (lane == 0 && k4_prefetch) {  // the warp's next slice on its way into L2 (TMA bulk prefetch)
            const long tn = t + (long)gridDim.x * nw;
            if (tn < tasks) {
                const long rn = tn / M;
                const long i0 = (tn - rn * M) * N, i1 = min(i0 + N, ir_len);
                const uintptr_t a = (reinterpret_cast<uintptr_t>(ir + rn * ir_stride + i0) + 15) & ~uintptr_t(15);
                const uintptr_t e = reinterpret_cast<uintptr_t>(ir + rn * ir_stride + i1) & ~uintptr_t(15);
                if (e > a)
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"((unsigned)(e - a))
                                 : "memory");
            }
        }
        auto load0 = [&](int, int n) -> float2 {  // z_n = (h[2n], h[2n+1])
            const long i0 = base + 2 * n;
            if (vec && i0 + 1 < ir_len) return __ldcs(reinterpret_cast<const float2*>(h + i0));
            return make_float2(i0 < ir_len ? h[i0] : 0.f, i0 + 1 < ir_len ? h[i0 + 1] : 0.f);
        };
        fft_warp4<false, N, true>(buf, tw + N, lane, load0);
        untangle_pairs_warp(buf, N, s_pk, pool + ((row0 + row) * M + m) * N, lane);
        __syncwarp();
    }
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    TL_END(1);
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

// Multi-GPU stereo mix over peer memory (C3), fused: each thread sums this GPU's
// sources for one (ear, sample) in source order (the mix_kernel order) and stores the partial
// straight into slot `rank` of every rank's gather buffer — its own and, over NVLink, the peers'
// (cudaIpc-mapped) — so the reduction's transfer is the kernel's own store stream.
__global__ void mix_scatter_kernel(long sources, long ears, long samples, const float* __restrict__ out,
                                   long out_stride, float* const* __restrict__ slots, int world, int rank,
                                   long cap) {
    const long total = ears * samples;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long e = i / samples, t = i % samples;
        float acc = 0.f;
        for (long s = 0; s < sources; ++s) acc += out[(s * ears + e) * out_stride + t];
        const long off = ((long)rank * ears + e) * cap + t;
        for (int r = 0; r < world; ++r) slots[r][off] = acc;
    }
}

// mix[e][t] = sum over ranks, in rank order, of the gathered partials: every rank computes the
// same sums in the same order, so the mix is bit-identical on all of them (deterministic, unlike
// a ring all-reduce whose summation order depends on the rank).
__global__ void mix_gather_kernel(long ears, long samples, const float* __restrict__ gather, int world, long cap,
                                  float* __restrict__ mix, long mix_stride) {
    const long total = ears * samples;
    for (long i = blockIdx.x * (long)blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const long e = i / samples, t = i % samples;
        float acc = gather[e * cap + t];
        for (int r = 1; r < world; ++r) acc += gather[((long)r * ears + e) * cap + t];
        mix[e * mix_stride + t] = acc;
    }
}

int grid_for(long work, int threads) {
    long b = (work + threads - 1) / threads;
    return (int)std::max<long>(1, std::min<long>(b, 148L * 16));
}

int fft_threads(int N) { return std::max(32, std::min(256, N / 4)); }


// ---------------------------------------------------------------- comparison convolvers (§8f row 4)
// OLA / OLS / WOLA (reference.cpp:182-320) on the TVOLAP building blocks with M = 1: one CTA per
// (channel, hop) frames the hop, takes the real 2B transform (B = block = IR length) as a B-point
// complex Stockham FFT + untangle, multiplies by the channel's filter spectrum (packed bins),
// tangles and inverse-transforms into a per-hop scratch frame (WOLA: synthesis window applied).
// Frames depend only on the inputs, so every hop of a call transforms in parallel; the tails are
// then combined across hops by fbconv_combine_kernel. kind: 2 ola, 3 ols, 4 wola.
__global__ void __launch_bounds__(256) fbconv_frames_kernel(int kind, int B, int n_hops, const float* __restrict__ in,
                                                            long in_stride, const float* __restrict__ prev,
                                                            const float2* __restrict__ spec,
                                                            const float* __restrict__ win,
                                                            const float2* __restrict__ tw,
                                                            const float2* __restrict__ pk, float* __restrict__ yhat) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int N = B;  // complex points of the real 2B transform
    const int c = blockIdx.y, j = blockIdx.x, tid = threadIdx.x, NT = blockDim.x;
    const int hop = kind == 4 ? B / 2 : B;
    float2* s_tw = reinterpret_cast<float2*>(smem);
    float2* s_pk = s_tw + N;
    float2* s_a = s_pk + N + 2;
    float2* s_b = s_a + N;
    for (int i = tid; i < N; i += NT) s_tw[i] = tw[i];
    for (int i = tid; i <= N; i += NT) s_pk[i] = pk[i];
    const float* x = in + (long)c * in_stride + (long)j * hop;  // this hop
    // the previous hop's input: the call's own previous hop, or the carried state for j = 0
    const float* xp = j > 0 ? x - hop : prev + (long)c * hop;
    auto frame = [&](int i) -> float {  // real frame sample i < 2B
        if (kind == 2) return i < B ? x[i] : 0.f;
        if (kind == 3) return i < B ? xp[i] : x[i - B];
        const int h = B / 2;
        if (i < h) return xp[i] * win[i];
        return i < B ? x[i - h] * win[i] : 0.f;
    };
    for (int k = tid; k < N; k += NT) s_a[k] = make_float2(frame(2 * k), frame(2 * k + 1));
    __syncthreads();
    const bool prune = kind != 3;  // OLA and WOLA frames are zero past B
    const float2* Z = fft_batch<false, 0>(s_a, s_b, N, 1, s_tw, prune, tid, NT);
    float2* Y = Z == s_a ? s_b : s_a;
    const float2* H = spec + (long)c * N;
    for (int k = tid; k < N; k += NT) {
        const float2 X = untangle_packed(Z, N, k, s_pk);
        const float2 h = H[k];
        Y[k] = k == 0 ? make_float2(X.x * h.x, X.y * h.y) : cmul(X, h);  // DC / Nyquist real (packed bin 0)
    }
    __syncthreads();
    float2* T = const_cast<float2*>(Z);
    for (int k = tid; k < N; k += NT) T[k] = tangle_packed(Y, N, k, s_pk);
    __syncthreads();
    const float2* yt = fft_batch<true, 0>(T, Y, N, 1, s_tw, false, tid, NT);
    const float sc = 1.0f / (float)N;
    float* o = yhat + ((long)c * n_hops + j) * 2 * B;
    for (int k = tid; k < N; k += NT) {
        float a = yt[k].x * sc, b = yt[k].y * sc;
        if (kind == 4 && 2 * k < B) {  // synthesis window over the block itself (reference.cpp:300-302)
            a *= win[2 * k];
            b *= win[2 * k + 1];
        }
        o[2 * k] = a;
        o[2 * k + 1] = b;
    }
}

// Tail combination across the hops of a call (one thread per (channel, sample of a hop)) and the
// carried state: OLA remainder [C][B]; OLS / WOLA previous input hop [C][hop]; WOLA three pending
// partial sums [C][3][hop] (the 2B accumulator of reference.cpp:304-307 shifted by one hop).
__global__ void fbconv_combine_kernel(int kind, int B, int channels, int n_hops, const float* __restrict__ in,
                                      long in_stride, const float* __restrict__ yhat, float* __restrict__ out,
                                      long out_stride, float* __restrict__ rem, float* __restrict__ prev) {
    const int hop = kind == 4 ? B / 2 : B;
    const long i = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long)channels * hop) return;
    const int c = (int)(i / hop), u = (int)(i % hop);
    const float* y = yhat + (long)c * n_hops * 2 * B;
    float* o = out + (long)c * out_stride;
    if (kind == 2) {
        float r = rem[(long)c * B + u];
        for (int j = 0; j < n_hops; ++j) {
            o[(long)j * hop + u] = y[(long)j * 2 * B + u] + r;
            r = y[(long)j * 2 * B + B + u];
        }
        rem[(long)c * B + u] = r;
    } else if (kind == 3) {
        for (int j = 0; j < n_hops; ++j) o[(long)j * hop + u] = y[(long)j * 2 * B + B + u];
    } else {
        float* A = rem + (long)c * 3 * hop;
        float a0 = A[u], a1 = A[hop + u], a2 = A[2 * hop + u];
        for (int j = 0; j < n_hops; ++j) {
            const float* yj = y + (long)j * 2 * B;
            o[(long)j * hop + u] = 0.5f * (a0 + yj[u]);
            a0 = a1 + yj[hop + u];
            a1 = a2 + yj[2 * hop + u];
            a2 = yj[3 * hop + u];
        }
        A[u] = a0;
        A[hop + u] = a1;
        A[2 * hop + u] = a2;
    }
    if (kind != 2) prev[(long)c * hop + u] = in[(long)c * in_stride + (long)(n_hops - 1) * hop + u];
}

// Direct-form FIR for "tdc" / "cf-tdc" (reference.cpp:68-93, 136-172): out[t] = sum_q h[q] xx[t+taps-1-q]
// over xx = [history (taps-1) | this call's samples]. The first `fade_len` samples of the call blend
// the old filter's output in with g_new = gain(fade_elapsed0 + t) (Hann-complementary or linear).
// One CTA = 256 consecutive outputs of one channel; taps are streamed through shared memory in
// chunks of kFirChunk together with the input span they touch.
constexpr int kFirTile = 256, kFirChunk = 512;
__global__ void __launch_bounds__(kFirTile) fir_kernel(int taps, long T, const float* __restrict__ xx, long xx_stride,
                                                       const float* __restrict__ h, const float* __restrict__ h_old,
                                                       float* __restrict__ out, long out_stride, long fade_len,
                                                       long fade_elapsed0, long fade_duration, int fade_shape) {
    __shared__ float s_h[kFirChunk], s_ho[kFirChunk], s_x[kFirTile + kFirChunk];
    const int c = blockIdx.y, tid = threadIdx.x;
    const long t0 = (long)blockIdx.x * kFirTile, t = t0 + tid;
    const bool blend_cta = t0 < fade_len;
    const float* xc = xx + (long)c * xx_stride;
    const float* hc = h + (long)c * taps;
    const float* hoc = h_old + (long)c * taps;
    float acc = 0.f, acc_old = 0.f;
    for (int q0 = 0; q0 < taps; q0 += kFirChunk) {
        const int qn = min(kFirChunk, taps - q0);
        __syncthreads();
        for (int k = tid; k < qn; k += kFirTile) {
            s_h[k] = hc[q0 + k];
            if (blend_cta) s_ho[k] = hoc[q0 + k];
        }
        // outputs t0 .. t0+255 with taps q0 .. q0+qn-1 read xx[t0 + taps-1-q0-(qn-1) .. t0+255 + taps-1-q0]
        const long base = t0 + taps - 1 - q0 - (qn - 1);
        for (int k = tid; k < kFirTile + qn - 1; k += kFirTile) {
            const long idx = base + k;
            s_x[k] = idx < T + taps - 1 ? xc[idx] : 0.f;
        }
        __syncthreads();
        if (t < T) {
            // xx index of (t, q) relative to base: tid + (qn - 1) - (q - q0)
            for (int k = 0; k < qn; ++k) {
                const float xv = s_x[tid + qn - 1 - k];
                acc = fmaf(s_h[k], xv, acc);
                if (blend_cta) acc_old = fmaf(s_ho[k], xv, acc_old);
            }
        }
    }
    if (t >= T) return;
    float y = acc;
    if (t < fade_len) {
        const long e = fade_elapsed0 + t;
        double g = 1.0;
        if (e < fade_duration && fade_duration != 1) {
            const double phase = (double)e / (double)fade_duration;
            g = fade_shape == 1 ? phase : 0.5 * (1.0 - cos(3.14159265358979323846 * phase));
        }
        y = (float)(1.0 - g) * acc_old + (float)g * acc;
    }
    out[(long)c * out_stride + t] = y;
}

}  // namespace

size_t hop_kernel_smem_bytes(int L, int P, int E, int qm) { return SmemLayout(L, P, E, qm).total; }

size_t block_kernel_smem_bytes(int L, int P, int E, int JH, bool bank, int threads) {
    return BlockLayout(L, P, E, 2 * JH, bank, threads).total;
}

template <int E, int JH, bool BANK>
static cudaError_t launch_block_t(const HopParams& p, int Q, int threads, cudaStream_t stream) {
    const size_t smem = block_kernel_smem_bytes(p.L, p.P, E, JH, BANK, threads);
    // compile-time transform length for the BASELINE geometries (and the one each kernel
    // variant actually serves), runtime N otherwise
    void (*fn)(const HopParams, const int) = tvolap_block_kernel<E, JH, BANK, 0>;
    const int N = 2 * p.L;
    if constexpr (!BANK && E == 1 && (JH == 4 || JH == 8)) {
        const bool sw = p.sw_count > 0;  // switching launches: the in-kernel K4 instantiation
        if (N == 256) fn = sw ? tvolap_block_kernel<E, JH, BANK, 256, true> : tvolap_block_kernel<E, JH, BANK, 256>;
        if (N == 512) fn = sw ? tvolap_block_kernel<E, JH, BANK, 512, true> : tvolap_block_kernel<E, JH, BANK, 512>;
        if (N == 1024) fn = sw ? tvolap_block_kernel<E, JH, BANK, 1024, true> : tvolap_block_kernel<E, JH, BANK, 1024>;
    }
    if constexpr (BANK && E == 1 && JH == 8) {
        if (N == 64) fn = tvolap_block_kernel<E, JH, BANK, 64>;
    }
    if constexpr (BANK && E == 2 && JH == 4) {
        if (N == 256) fn = tvolap_block_kernel<E, JH, BANK, 256>;
    }
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
    cudaLaunchAttribute attr[2];
    unsigned na = 0;
    if (p.P > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = (unsigned)p.P;
        attr[na].val.clusterDim.y = 1;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    if (g_launch_pdl) {  // tuning "pdl" (A/B: profiles/r01_ab_pdl.txt)  // overlap this launch's setup with the previous hop launch's tail
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, fn, p, Q);
}

cudaError_t launch_block_kernel(const HopParams& p, int E, int JH, int Q, int threads, cudaStream_t stream) {
    if (p.sched == nullptr && E == 1) {
        switch (JH) {
            case 1: return launch_block_t<1, 1, false>(p, Q, threads, stream);
            case 2: return launch_block_t<1, 2, false>(p, Q, threads, stream);
            case 4: return launch_block_t<1, 4, false>(p, Q, threads, stream);
            default: return launch_block_t<1, 8, false>(p, Q, threads, stream);
        }
    }
    if (E == 2) {
        switch (JH) {
            case 1: return launch_block_t<2, 1, true>(p, Q, threads, stream);
            case 2: return launch_block_t<2, 2, true>(p, Q, threads, stream);
            case 4: return launch_block_t<2, 4, true>(p, Q, threads, stream);
            default: return launch_block_t<2, 8, true>(p, Q, threads, stream);
        }
    }
    switch (JH) {
        case 1: return launch_block_t<1, 1, true>(p, Q, threads, stream);
        case 2: return launch_block_t<1, 2, true>(p, Q, threads, stream);
        case 4: return launch_block_t<1, 4, true>(p, Q, threads, stream);
        default: return launch_block_t<1, 8, true>(p, Q, threads, stream);
    }
}

namespace {
// ring geometry (steps per stage R, stages ST) by variant v = HopParams::ring_var: sized so that
// several CTAs share an SM (their transforms overlap each other's MACs) with ~100 KB of rows in
// flight per SM
__host__ __device__ constexpr int ring_r(int N, int v) {
    return N == 64 ? (v == 2 ? 8 : v == 4 ? 2 : 4) : (v >= 3 ? 4 : 2);
}
__host__ __device__ constexpr int ring_st(int N, int v) {
    return N == 64 ? (v >= 3 ? 4 : 3) : (v == 1 || v == 4 ? 3 : 2);
}

template <int E, int NC, int VAR>
cudaError_t launch_hop_ring_t(const HopParams& p, int threads, cudaStream_t stream) {
    constexpr int R = ring_r(NC, VAR), ST = ring_st(NC, VAR);
    auto fn = tvolap_hop_ring_kernel<E, NC, R, ST>;
    const size_t smem = RingLayout(p.L, E, p.qm, R, ST).total;
    cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem)) != cudaSuccess) return err;
    fn<<<(unsigned)std::min<long>(p.S, (long)sms * std::max(1, per_sm)), threads, smem, stream>>>(p);
    return cudaGetLastError();
}
template <int E, int NC>
cudaError_t launch_hop_ring_v(const HopParams& p, int threads, cudaStream_t stream) {
    switch (p.ring_var) {
        case 2: return launch_hop_ring_t<E, NC, 2>(p, threads, stream);
        case 3: return launch_hop_ring_t<E, NC, 3>(p, threads, stream);
        case 4: return launch_hop_ring_t<E, NC, 4>(p, threads, stream);
        default: return launch_hop_ring_t<E, NC, 1>(p, threads, stream);
    }
}
}  // namespace

// The ring kernel covers: bank engines (a latched selection), one hop, P = 1, 64- or 256-point
// spectra, one float4 column of one partition group per thread, whole stages per group.
bool hop_ring_supported(const HopParams& p, int E, int threads) {
    const int N = 2 * p.L, G = p.qm;
    if (!(N == 64 || N == 256) || p.P != 1 || p.n_hops != 1 || !p.sched || p.new_ir || G < 1) return false;
    if (threads != G * p.L || p.M % G || p.ring_var < 1 || p.ring_var > 4) return false;
    const int R = ring_r(N, p.ring_var), ST = ring_st(N, p.ring_var);
    const int MG = p.M / G;
    if (MG % R || MG / R < ST || p.D < R) return false;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (p.S > (long)kRingSources * sms) return false;  // the per-CTA source table
    return RingLayout(p.L, E, G, R, ST).total <= 227 * 1024;
}

cudaError_t launch_hop_ring_kernel(const HopParams& p, int E, int threads, cudaStream_t stream) {
    if (!hop_ring_supported(p, E, threads)) return cudaErrorInvalidValue;
    if (2 * p.L == 64) return E == 2 ? launch_hop_ring_v<2, 64>(p, threads, stream) : launch_hop_ring_v<1, 64>(p, threads, stream);
    return E == 2 ? launch_hop_ring_v<2, 256>(p, threads, stream) : launch_hop_ring_v<1, 256>(p, threads, stream);
}

cudaError_t launch_hop_kernel(const HopParams& p, int E, int threads, cudaStream_t stream) {
    const size_t smem = hop_kernel_smem_bytes(p.L, p.P, E, p.qm);
    void (*fn)(const HopParams) = nullptr;
#define TV_HOP(NCV) fn = E == 2 ? tvolap_hop_kernel<2, NCV> : tvolap_hop_kernel<1, NCV>
    switch (2 * p.L) {
        case 64: TV_HOP(64); break;
        case 256: TV_HOP(256); break;
        case 512: TV_HOP(512); break;
        case 1024: TV_HOP(1024); break;
        default: TV_HOP(0);
    }
#undef TV_HOP
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

template <int NC>
static cudaError_t launch_partition_warp(int M, long rows, const float* ir, long ir_stride, long ir_len,
                                        float2* pool, long row0, const float2* tw, const float2* pk,
                                        cudaStream_t stream, bool pdl) {
    constexpr int kWarps = 8;
    const size_t smem = align16((2 * NC + 2) * sizeof(float2)) + (size_t)kWarps * NC * sizeof(float2);
    cudaError_t err = cudaFuncSetAttribute(partition_warp_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, partition_warp_kernel<NC>, 32 * kWarps, smem);
    if (err != cudaSuccess) return err;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long tasks = rows * M;
    const long grid = std::max<long>(1, std::min<long>((tasks + kWarps - 1) / kWarps, (long)sms * std::max(1, per_sm)));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(32 * kWarps);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, partition_warp_kernel<NC>, M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk,
                              (int)g_launch_k4_prefetch);  // tuning "k4_prefetch": per-slice L2 prefetch
}

cudaError_t launch_partition(int L, int M, long rows, const float* ir, long ir_stride, long ir_len, float2* pool,
                             long row0, const float2* tw, const float2* pk, cudaStream_t stream, bool pdl) {
    // one warp per partition for the common transform lengths (tuning "k4_warp" = 0: CTA batches)
    if (g_launch_k4_warp) {
        switch (2 * L) {
            case 64: return launch_partition_warp<64>(M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk, stream, pdl);
            case 128: return launch_partition_warp<128>(M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk, stream, pdl);
            case 256: return launch_partition_warp<256>(M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk, stream, pdl);
            case 512: return launch_partition_warp<512>(M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk, stream, pdl);
            case 1024: return launch_partition_warp<1024>(M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk, stream, pdl);
            default: break;
        }
    }
    // Batches of up to 8 partitions per CTA, 16-byte IR loads: enough bytes in flight to
    // stream the time-domain IRs near HBM speed.
    const int N = 2 * L;
    const long tasks = rows * M;
    // ~56 KB of shared memory per CTA (tables + two batch buffers): 4 CTAs per SM stay resident
    const long budget = 56L * 1024 - 16L * N;
    const int nf = (int)std::max<long>(1, std::min<long>({8L, tasks, budget / (16L * N)}));
    const int threads = std::max(32, std::min(256, nf * N / 8));
    const size_t smem = (size_t)(2 * N + 2 + 2 * (size_t)nf * N) * sizeof(float2);
    decltype(&partition_kernel<0>) fn = partition_kernel<0>;
    switch (N) {
        case 64: fn = partition_kernel<64>; break;
        case 256: fn = partition_kernel<256>; break;
        case 512: fn = partition_kernel<512>; break;
        case 1024: fn = partition_kernel<1024>; break;
        default: break;
    }
    cudaError_t err = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    const int grid = (int)std::max<long>(1, std::min<long>((tasks + nf - 1) / nf, 148L * 4));
    fn<<<grid, threads, smem, stream>>>(L, M, rows, ir, ir_stride, ir_len, pool, row0, tw, pk, nf);
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

cudaError_t launch_mix_scatter(long sources, long ears, long samples, const float* out, long out_stride,
                               float* const* slots, int world, int rank, long cap, cudaStream_t stream) {
    mix_scatter_kernel<<<grid_for(ears * samples, 256), 256, 0, stream>>>(sources, ears, samples, out, out_stride,
                                                                         slots, world, rank, cap);
    return cudaGetLastError();
}

cudaError_t launch_mix_gather(long ears, long samples, const float* gather, int world, long cap, float* mix,
                              long mix_stride, cudaStream_t stream) {
    mix_gather_kernel<<<grid_for(ears * samples, 256), 256, 0, stream>>>(ears, samples, gather, world, cap, mix,
                                                                        mix_stride);
    return cudaGetLastError();
}

cudaError_t launch_fbconv(int kind, int B, long channels, long n_hops, const float* in, long in_stride, float* prev,
                          const float2* spec, const float* win, const float2* tw, const float2* pk, float* yhat,
                          float* out, long out_stride, float* rem, cudaStream_t stream) {
    const size_t smem = (size_t)(4 * (size_t)B + 2) * sizeof(float2);
    cudaError_t err = cudaFuncSetAttribute(fbconv_frames_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err != cudaSuccess) return err;
    fbconv_frames_kernel<<<dim3((unsigned)n_hops, (unsigned)channels), 256, smem, stream>>>(kind, B, (int)n_hops, in,
                                                                                          in_stride, prev, spec, win, tw,
                                                                                          pk, yhat);
    err = cudaGetLastError();
    if (err != cudaSuccess) return err;
    const long hop = kind == 4 ? B / 2 : B;
    fbconv_combine_kernel<<<grid_for(channels * hop, 256), 256, 0, stream>>>(kind, B, (int)channels, (int)n_hops, in,
                                                                            in_stride, yhat, out, out_stride, rem, prev);
    return cudaGetLastError();
}

cudaError_t launch_fir(int taps, long channels, long T, const float* xx, long xx_stride, const float* h,
                       const float* h_old, float* out, long out_stride, long fade_len, long fade_elapsed0,
                       long fade_duration, int fade_shape, cudaStream_t stream) {
    const dim3 grid((unsigned)((T + kFirTile - 1) / kFirTile), (unsigned)channels);
    fir_kernel<<<grid, kFirTile, 0, stream>>>(taps, T, xx, xx_stride, h, h_old, out, out_stride, fade_len,
                                              fade_elapsed0, fade_duration, fade_shape);
    return cudaGetLastError();
}

}  // namespace tvb

#ifdef TVOLAP_PHASE_PROF
extern "C" int tvolap_phase_counters(unsigned long long* out, int n) {
    unsigned long long zero[16] = {};
    n = n < 16 ? n : 16;
    if (cudaDeviceSynchronize() != cudaSuccess) return 6;
    if (cudaMemcpyFromSymbol(out, g_phase, n * sizeof(unsigned long long)) != cudaSuccess) return 6;
    return cudaMemcpyToSymbol(g_phase, zero, sizeof(zero)) == cudaSuccess ? 0 : 6;
}

// timeline: out[kind][i][2] for the first `n` launches of each kind since the last reset
extern "C" int tvolap_timeline(unsigned long long* out, int n, unsigned* counts) {
    if (cudaDeviceSynchronize() != cudaSuccess) return 6;
    if (cudaMemcpyFromSymbol(counts, g_tl_n, 2 * sizeof(unsigned)) != cudaSuccess) return 6;
    static unsigned long long tmp[2][4096][2];
    if (cudaMemcpyFromSymbol(tmp, g_tl, sizeof(tmp)) != cudaSuccess) return 6;
    n = n < 4096 ? n : 4096;
    for (int k = 0; k < 2; ++k)
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < 2; ++j) out[(k * n + i) * 2 + j] = tmp[k][i][j];
    const unsigned zero[2] = {0, 0};
    return cudaMemcpyToSymbol(g_tl_n, zero, sizeof(zero)) == cudaSuccess ? 0 : 6;
}
#endif
