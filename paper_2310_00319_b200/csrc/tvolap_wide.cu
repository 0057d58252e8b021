// Time-parallel ("wide") pass of the TVOLAP engine for long device-resident calls.
//
// A call that carries all of its hops (tvolap_process_switching on device buffers) fixes every
// input frame and every filter set up front, so nothing in the per-hop pipeline of
// proj/src/engine.cpp:60-106 is sequential across hops except the hop-2 overlap-add carry
// (engine.cpp:97-102), which is a 3-value linear recurrence per output sample. The hop-blocked
// kernel walks the hops of a lane in order (parallelism = lanes x cluster CTAs: 256 CTAs for
// C2); here the hop axis is parallel too:
//   wide_head_kernel          the spectra of hops before the call (still needed by its first
//                             outputs) from the delay line into the extended spectra buffer Xe,
//   wide_forward[_warp]_kernel K1 for every hop of the call at once (window + pruned FFT +
//                             untangle), into Xe; the last 2D hops also into the delay line,
//   partition_multi_kernel    K4 for every filter set of the call (periods longer than a tile),
//   wide_mac_kernel           one CTA per (lane, tile of <= 16 hops inside one filter period):
//                             K4 of the period's set into an L2 scratch slot (periods of one
//                             tile), K3 over Xe with a sliding register window, then K5 (tangle
//                             + inverse FFT) and the overlap-add of the tile's outputs from its
//                             4th hop on,
//   wide_fixup_kernel         the first three outputs of every tile from the carry of the tile
//                             before it (and the engine's carry / history for the next call).
// The MAC sums the partition groups in the hop-blocked kernel's order and the OLA recurrence runs
// in the sequential order. With the hop kernels' CTA Stockham transforms for K1/K5
// (TVOLAP_WIDE_WARPFFT=0) the outputs are bit-identical to tvolap_block_kernel's; the default
// warp-per-frame transforms (fft_warp4) equal them to fp32 rounding (tests/test_gpu_wide.py).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <utility>

#include "tvolap_fft.cuh"
#include "tvolap_internal.cuh"

namespace tvb {
namespace {

__host__ __device__ inline size_t a16(size_t x) { return (x + 15) & ~size_t(15); }


// Delay-line history of the call: Xe[s][parity][t] holds the spectrum of hop j with
// j & 1 == parity and t = (j >> 1) - tbase, for every hop the call's outputs read.
__global__ void wide_head_kernel(const WideParams p) {
    const int N = 2 * p.L, V = N / 2;
    const int nh = p.M + 2 + kWideFront;  // slots per parity that can precede hop0
    const long total = (long)p.S * 2 * nh * V;
    const float4* ring4 = reinterpret_cast<const float4*>(p.ring);
    float4* xe4 = reinterpret_cast<float4*>(p.xe);
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int v = (int)(i % V);
        const long r = i / V;
        const int t = (int)(r % nh);
        const int par = (int)((r / nh) & 1);
        const long s = r / (2 * nh);
        const long j = 2 * (t + p.tbase) + par;  // hop held in this slot
        if (j >= p.hop0) continue;               // written by wide_forward_kernel
        float4 val = make_float4(0.f, 0.f, 0.f, 0.f);
        if (j >= 0) {
            const long slot = (j >> 1) % p.D;
            val = ring4[((s * 2 + par) * p.D + slot) * V + v];
        }
        xe4[((s * 2 + par) * p.T + t) * V + v] = val;
    }
}

// K1 for every hop of the pass (engine.cpp:77-82): the operations of the hop-blocked kernel's
// forward phase (window products, fft_batch, untangle_store). Persistent CTAs walk work items
// (lane, kFwdF consecutive frames); the raw input of the next item (kFwdF + 1 hops, the first
// one being the previous hop) is loaded into registers while the current item's FFTs run.
constexpr int kFwdF = 4;

template <int NC>
__global__ void __launch_bounds__(256) wide_forward_kernel(const WideParams p) {
    constexpr int N = NC, L = NC / 2, F = kFwdF, SPAN = (F + 1) * L, PER = (SPAN + 255) / 256;
    extern __shared__ __align__(16) unsigned char smem[];
    float2* s_tw = reinterpret_cast<float2*>(smem);
    float2* s_pk = reinterpret_cast<float2*>(smem + a16(N * sizeof(float2)));
    float* s_win = reinterpret_cast<float*>(smem + a16(N * sizeof(float2)) + a16((N + 2) * sizeof(float2)));
    float* s_x = reinterpret_cast<float*>(reinterpret_cast<unsigned char*>(s_win) + a16(N * sizeof(float)));
    float2* s_fa = reinterpret_cast<float2*>(reinterpret_cast<unsigned char*>(s_x) + a16(SPAN * sizeof(float)));
    float2* s_fb = s_fa + (size_t)F * N;
    const int tid = threadIdx.x, NT = 256;
    for (int i = tid; i < N; i += NT) {
        s_tw[i] = p.tw[i];
        s_win[i] = p.win[i];
    }
    for (int i = tid; i <= N; i += NT) s_pk[i] = p.pk[i];
    const int chunks = (p.n + F - 1) / F;
    const long items = (long)p.S * chunks;
    // raw samples of item w: hops r0 - 1 .. r0 + F - 1 (hop -1 of the pass = the history)
    auto load = [&](long w, float (&v)[PER]) {
        const long s = w / chunks;
        const int r0 = (int)(w - s * chunks) * F;
        const float* xin = p.in + s * p.in_stride;
#pragma unroll
        for (int c = 0; c < PER; ++c) {
            const int i = tid + c * NT;
            const int r = r0 - 1 + i / L;  // hop of the pass
            float val = 0.f;
            if (i < SPAN && r < p.n) val = r < 0 ? p.hist[s * L + (i % L)] : __ldcs(xin + (long)r * L + (i % L));
            v[c] = val;
        }
    };
    float v[PER];
    long w = blockIdx.x;
    if (w < items) load(w, v);
    const long ring_from = p.hop0 + p.n - 2L * p.D;  // these hops stay in the delay line after the call
    for (; w < items; w += gridDim.x) {
        const long s = w / chunks;
        const int r0 = (int)(w - s * chunks) * F;
        const int nf = min(F, p.n - r0);
        __syncthreads();  // previous item's FFT buffers and s_x are free (and the tables loaded)
#pragma unroll
        for (int c = 0; c < PER; ++c)
            if (tid + c * NT < SPAN) s_x[tid + c * NT] = v[c];
        if (w + gridDim.x < items) load(w + gridDim.x, v);  // in flight during this item's FFTs
        __syncthreads();
        for (int i = tid; i < nf * L; i += NT) {
            const int f = i / L, jj = i - f * L;
            const float* xs = s_x + f * L;  // (hop r0 + f - 1 | hop r0 + f)
            s_fa[(size_t)f * N + jj] = make_float2(xs[2 * jj] * s_win[2 * jj], xs[2 * jj + 1] * s_win[2 * jj + 1]);
        }
        __syncthreads();
        const float2* Z = fft_batch<false, NC>(s_fa, s_fb, N, nf, s_tw, true, tid, NT);
        for (int f = 0; f < nf; ++f) {
            const long j = p.hop0 + r0 + f;
            const int par = (int)(j & 1);
            float2* dst = p.xe + ((s * 2 + par) * p.T + ((j >> 1) - p.tbase)) * N;
            untangle_store<NC>(Z + (size_t)f * N, N, s_pk, dst, tid, NT);
            if (j >= ring_from)
                untangle_store<NC>(Z + (size_t)f * N, N, s_pk, p.ring + ((s * 2 + par) * p.D + (j >> 1) % p.D) * N,
                                   tid, NT);
        }
    }
}

// K1 with one warp per frame (warp four-step FFT, no CTA barriers): frame f = (lane f / n,
// hop f mod n), lane-major so consecutive warps share input hops. Same values as the Stockham
// K1 up to fp32 rounding (a different factorisation).
template <int NC>
__global__ void __launch_bounds__(256) wide_forward_warp_kernel(const WideParams p) {
    constexpr int N = NC, L = NC / 2;
    extern __shared__ __align__(16) unsigned char smem[];
    float2* s_pk = reinterpret_cast<float2*>(smem);
    float* s_win = reinterpret_cast<float*>(smem + a16((N + 2) * sizeof(float2)));
    float2* bufs = reinterpret_cast<float2*>(reinterpret_cast<unsigned char*>(s_win) + a16(N * sizeof(float)));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    for (int i = tid; i < N; i += blockDim.x) s_win[i] = p.win[i];
    for (int i = tid; i <= N; i += blockDim.x) s_pk[i] = p.pk[i];
    __syncthreads();
    // two frames per warp in lockstep (independent FFT chains): pairs (2q, 2q + 1) of the
    // lane-major frame order; a lone last frame is computed twice and stored once
    float2* buf = bufs + (size_t)warp * 2 * N;
    const long frames = (long)p.S * p.n;
    const long pairs = (frames + 1) / 2;
    const long ring_from = p.hop0 + p.n - 2L * p.D;
    for (long q = (long)blockIdx.x * nw + warp; q < pairs; q += (long)gridDim.x * nw) {
        const float* prev[2];
        const float* cur[2];
        long sf[2], jf[2];
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const long f = min(2 * q + t, frames - 1);
            const long s = f / p.n;
            const int r = (int)(f - s * p.n);
            prev[t] = r == 0 ? p.hist + s * L : p.in + s * p.in_stride + (long)(r - 1) * L;
            cur[t] = p.in + s * p.in_stride + (long)r * L;
            sf[t] = s;
            jf[t] = p.hop0 + r;
        }
        auto load2 = [&](int t, int n) -> float2 {  // z_n = (x[2n] w[2n], x[2n+1] w[2n+1]), n < L
            const int e = 2 * n;
            const float* src = e < L ? prev[t] + e : cur[t] + (e - L);
            return make_float2(src[0] * s_win[e], src[1] * s_win[e + 1]);
        };
        fft_warp4<false, N, true, 2>(buf, p.tw + N, lane, load2);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            if (2 * q + t >= frames) break;
            const long j = jf[t], s = sf[t];
            const int par = (int)(j & 1);
            untangle_pairs_warp(buf + (size_t)t * N, N, s_pk, p.xe + ((s * 2 + par) * p.T + ((j >> 1) - p.tbase)) * N,
                                lane);
            if (j >= ring_from)
                untangle_pairs_warp(buf + (size_t)t * N, N, s_pk,
                                    p.ring + ((s * 2 + par) * p.D + (j >> 1) % p.D) * N, lane);
        }
        __syncwarp();
    }
}

// K1 for 64-point transforms (L = 32: C5), where one warp per frame leaves two points per lane
// and the transform is all shuffles and index arithmetic (2.4 us per C5 hop against 0.4 us of
// memory time). Here 8 lanes own a frame (4 frames per warp, 32 consecutive hops of one source
// per CTA iteration): lane t holds z[8 n1 + t], an 8-point DFT in registers (upper half zero),
// twiddles W_64^(t k1), an 8 x 8 transpose through shared memory (row stride 9, frame stride 72
// float2: conflict-free), a second 8-point DFT, the spectrum left in natural order, then every
// lane untangles 8 bins and stores them as four float4 (spectral.cpp:105-124). Window, twiddles
// and pack phasors are per-lane constants held in registers.
__global__ void __launch_bounds__(256) wide_forward_small_kernel(const WideParams p) {
    constexpr int N = 64, L = 32, FS = 72;
    __shared__ __align__(16) float2 s_buf[8][4 * FS];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, t = lane & 7, fr = lane >> 3;
    float2* buf = s_buf[warp] + fr * FS;
    float2 wn[4], twr[8], pkr[8];
#pragma unroll
    for (int n1 = 0; n1 < 4; ++n1) wn[n1] = make_float2(p.win[2 * (8 * n1 + t)], p.win[2 * (8 * n1 + t) + 1]);
    twr[0] = make_float2(1.f, 0.f);
#pragma unroll
    for (int k1 = 1; k1 < 8; ++k1) {  // W_64^(t k1) from the four-step table (W_64^j, j < 32)
        const int j = t * k1;
        const float2 w = p.tw[N + 32 + (j & 31)];
        twr[k1] = (j & 32) ? make_float2(-w.x, -w.y) : w;
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        pkr[2 * i] = p.pk[2 * (t + 8 * i)];
        pkr[2 * i + 1] = p.pk[2 * (t + 8 * i) + 1];
    }
    const long ring_from = p.hop0 + p.n - 2L * p.D;
    const int chunks = (p.n + 31) / 32;
    const long items = (long)p.S * chunks;
    for (long it = blockIdx.x; it < items; it += gridDim.x) {
        const long s = it / chunks;
        const int r = (int)(it - s * chunks) * 32 + warp * 4 + fr;
        const bool valid = r < p.n;
        const int rc = min(r, p.n - 1);
        const float* cur = p.in + s * p.in_stride + (long)rc * L;
        const float* prev = rc == 0 ? p.hist + s * L : cur - L;
        float2 v[8];
#pragma unroll
        for (int n1 = 0; n1 < 4; ++n1) {  // z_n = (x[2n] w[2n], x[2n+1] w[2n+1]), n = 8 n1 + t < L
            const float* src = (n1 < 2 ? prev : cur - L) + 2 * (8 * n1 + t);
            v[n1] = make_float2(src[0] * wn[n1].x, src[1] * wn[n1].y);
            v[n1 + 4] = make_float2(0.f, 0.f);
        }
        dft_reg<false, 8, true>(v);
#pragma unroll
        for (int k1 = 1; k1 < 8; ++k1) v[k1] = twmul<false>(v[k1], twr[k1]);
#pragma unroll
        for (int k1 = 0; k1 < 8; ++k1) buf[k1 * 9 + t] = v[k1];
        __syncwarp();
#pragma unroll
        for (int n2 = 0; n2 < 8; ++n2) v[n2] = buf[t * 9 + n2];
        dft_reg<false, 8>(v);
        __syncwarp();
#pragma unroll
        for (int k2 = 0; k2 < 8; ++k2) buf[t + 8 * k2] = v[k2];  // Z[k1 + 8 k2], natural order
        __syncwarp();
        const long j = p.hop0 + rc;
        const int par = (int)(j & 1);
        float4* dst = reinterpret_cast<float4*>(p.xe + ((s * 2 + par) * p.T + ((j >> 1) - p.tbase)) * N);
        float4* rdst = j >= ring_from ? reinterpret_cast<float4*>(p.ring + ((s * 2 + par) * p.D + (j >> 1) % p.D) * N)
                                      : nullptr;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int j4 = t + 8 * i, k = 2 * j4;
            float2 a, b;
            {
                const float2 zk = buf[k], zm = buf[(N - k) & (N - 1)];
                if (k == 0) {
                    a = make_float2(zk.x + zk.y, zk.x - zk.y);
                } else {
                    const float2 even = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
                    const float2 odd = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
                    a = cadd(even, cmul(pkr[2 * i], odd));
                }
            }
            {
                const float2 zk = buf[k + 1], zm = buf[N - k - 1];
                const float2 even = make_float2(0.5f * (zk.x + zm.x), 0.5f * (zk.y - zm.y));
                const float2 odd = make_float2(0.5f * (zk.y + zm.y), -0.5f * (zk.x - zm.x));
                b = cadd(even, cmul(pkr[2 * i + 1], odd));
            }
            if (valid) {
                const float4 o = make_float4(a.x, a.y, b.x, b.y);
                dst[j4] = o;
                if (rdst) rdst[j4] = o;
            }
        }
        __syncwarp();
    }
}

// K4 for the sets a call installs: row r = k * S + s transforms irs[k] + s * ir_len into
// pool[(r * M + m) * N] (partition.cpp:20-51). Same warp transform as partition_warp_kernel.
template <int NC>
__global__ void __launch_bounds__(256, NC >= 1024 ? 2 : 3) partition_multi_kernel(int M, int S, long rows,
                                                                 const float* const* __restrict__ irs, long ir_len,
                                                                 float2* __restrict__ pool,
                                                                 const float2* __restrict__ tw,
                                                                 const float2* __restrict__ pk) {
    constexpr int N = NC;
    extern __shared__ __align__(16) unsigned char smem[];
    float2* s_pk = reinterpret_cast<float2*>(smem);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
    float2* buf = reinterpret_cast<float2*>(smem + a16((N + 2) * sizeof(float2))) + (size_t)warp * N;
    for (int i = tid; i <= N; i += blockDim.x) s_pk[i] = pk[i];
    __syncthreads();
    const long tasks = rows * M;
    for (long t = (long)blockIdx.x * nw + warp; t < tasks; t += (long)gridDim.x * nw) {
        const long row = t / M;
        const int m = (int)(t - row * M);
        const float* h = irs[row / S] + (row % S) * ir_len;
        const bool vec = (ir_len & 1) == 0 && (reinterpret_cast<uintptr_t>(h) & 7) == 0;
        const long base = (long)m * N;
        auto load0 = [&](int, int n) -> float2 {
            const long i0 = base + 2 * n;
            if (vec && i0 + 1 < ir_len) return __ldcs(reinterpret_cast<const float2*>(h + i0));
            return make_float2(i0 < ir_len ? h[i0] : 0.f, i0 + 1 < ir_len ? h[i0 + 1] : 0.f);
        };
        fft_warp4<false, N, true>(buf, tw + N, lane, load0);
        untangle_pairs_warp(buf, N, s_pk, pool + (row * M + m) * N, lane);
        __syncwarp();
    }
}

constexpr int kWideFB = 4;  // frames per inverse-FFT batch


struct WideLayout {
    size_t tw, pk, y, fa, fb, aux, total;
    __host__ __device__ WideLayout(int N, int J, int M, int Q) {
        tw = 0;
        pk = a16(tw + N * sizeof(float2));
        y = a16(pk + (N + 2) * sizeof(float2));
        fa = a16(y + (size_t)J * N * sizeof(float2));
        fb = a16(fa + (size_t)kWideFB * N * sizeof(float2));
        aux = a16(fb + (size_t)kWideFB * N * sizeof(float2));  // bin-0 Nyquist chains (K3)
        total = a16(aux + (size_t)(3 * M + J + Q * J) * sizeof(float));
    }
};

// K3 + K5 for one tile (lane blockIdx.y, hops tile0[x] .. tile0[x+1] of the call, one filter set):
//   Y_l = sum_m H[m] X_{l-2m} (engine.cpp:85-92) for every packed bin, the partitions in Q
//   contiguous groups summed in group order (the blocked kernel's grouping), then the inverse
//   real FFT (spectral.cpp:127-158) and the hop-2 overlap-add (engine.cpp:94-102).
template <int NC, int JH>
__global__ void __launch_bounds__(256, 2) wide_mac_kernel(const WideParams p) {
    constexpr int N = NC, L = NC / 2, J = 2 * JH;
    extern __shared__ __align__(16) unsigned char smem[];
    const WideLayout lay(N, J, p.M, p.Q);
    float2* s_tw = reinterpret_cast<float2*>(smem + lay.tw);
    float2* s_pk = reinterpret_cast<float2*>(smem + lay.pk);
    float2* s_y = reinterpret_cast<float2*>(smem + lay.y);
    float2* s_fa = reinterpret_cast<float2*>(smem + lay.fa);
    float2* s_fb = reinterpret_cast<float2*>(smem + lay.fb);
    const int tid = threadIdx.x, NT = blockDim.x;
    const int tile = blockIdx.x;
    const long s = blockIdx.y;
    const int l0r = p.tile0[tile], jt = p.tile0[tile + 1] - l0r;
    const long l0 = p.hop0 + l0r;
    const int M = p.M, Q = p.Q;
    for (int i = tid; i < N; i += NT) s_tw[i] = p.tw[i];
    for (int i = tid; i <= N; i += NT) s_pk[i] = p.pk[i];

    // ---- K4 fused (passes with one tile per filter period): the tile transforms its own set
    // (one warp per partition, the warp transform of partition_warp_kernel, bit-identical) into
    // a scratch slot held by this CTA; the slot stays in L2 and the MAC reads it straight back,
    // so the set's spectra never go to HBM. Slots: one per resident CTA, taken by atomicCAS.
    // The probe loop is bounded: nslots = max resident CTAs per SM x the device's SMs, a CTA takes
    // a slot only once it is resident and frees it before it retires, so fewer than nslots slots are
    // held whenever a CTA probes (fewer SMs under MPS / green contexts only lower the count); the
    // walk from its SM's home slot finds a free one within nslots probes. (A persistent-CTA variant
    // that owns slot blockIdx.x measured 9 % slower on C2: the item loop spills 116 B.)
    const float* tir = p.tile_ir ? p.tile_ir[tile] : nullptr;
    __shared__ int s_slot;
    int slot = -1;
    const float2* H = nullptr;
    if (tir) {
        if (tid == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            int sl = (int)((sm * 2u) % (unsigned)p.nslots);
            while (atomicCAS(p.slot_lock + sl, 0u, 1u) != 0u) sl = sl + 1 == p.nslots ? 0 : sl + 1;
            s_slot = sl;
        }
        __syncthreads();  // slot chosen, tables loaded
        slot = s_slot;
        float2* Hs = p.scratch + (size_t)slot * (M + kWideTail) * N;
        const float* h = tir + s * p.ir_len;
        const bool vec = (p.ir_len & 1) == 0 && (reinterpret_cast<uintptr_t>(h) & 7) == 0;
        const int lane = tid & 31, warp = tid >> 5, nw = NT >> 5;
        auto loader = [&](int m) {
            return [&, m](int, int n) -> float2 {
                const long i0 = (long)m * N + 2 * n;
                if (m >= M) return make_float2(0.f, 0.f);
                if (vec && i0 + 1 < p.ir_len) return __ldcs(reinterpret_cast<const float2*>(h + i0));
                return make_float2(i0 < p.ir_len ? h[i0] : 0.f, i0 + 1 < p.ir_len ? h[i0 + 1] : 0.f);
            };
        };
        // warp buffers in s_y (idle until the MAC's first group ends); same-box A/B: two partitions
        // per warp in lockstep (fft_warp4 NB = 2) spills and measured 6.24 vs 5.83 ms per C2 pass
        float2* buf = s_y + (size_t)warp * N;
        const bool staged = p.stage_ir && J >= 16 && p.ir_len >= (long)M * N && (p.ir_len & 3) == 0 &&
                            (reinterpret_cast<uintptr_t>(h) & 15) == 0;
        if (staged) {
            // IR slices (N floats) through a per-warp double buffer in rows 8..15 of s_y, one
            // partition ahead with 16-byte cp.async: the transform's loads hit shared memory
            float* pb = reinterpret_cast<float*>(s_y + (size_t)8 * N) + (size_t)warp * 2 * N;
            auto issue = [&](int m, int b) {
                if (m < M)
                    for (int i = 4 * lane; i < N; i += 128) {
                        const unsigned sa = (unsigned)__cvta_generic_to_shared(pb + (size_t)b * N + i);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(h + (long)m * N + i)
                                     : "memory");
                    }
                asm volatile("cp.async.commit_group;\n" ::: "memory");
            };
            int b = 0;
            issue(warp, 0);
            for (int m = warp; m < M; m += nw, b ^= 1) {
                issue(m + nw, b ^ 1);
                asm volatile("cp.async.wait_group 1;\n" ::: "memory");
                __syncwarp();
                const float* cur = pb + (size_t)b * N;
                fft_warp4<false, N, true>(buf, p.tw + N, lane,
                                          [&](int, int n) { return make_float2(cur[2 * n], cur[2 * n + 1]); });
                untangle_pairs_warp(buf, N, s_pk, Hs + (long)m * N, lane);
                __syncwarp();
            }
            asm volatile("cp.async.wait_all;\n" ::: "memory");
        } else {
            for (int m = warp; m < M; m += nw) {
                fft_warp4<false, N, true>(buf, p.tw + N, lane, loader(m));
                untangle_pairs_warp(buf, N, s_pk, Hs + (long)m * N, lane);
                __syncwarp();
            }
        }
        __syncthreads();  // the set's spectra (global, this CTA's writes) visible to all its threads
        H = Hs;
    } else {
        H = p.fset_per_lane ? p.fset[(long)tile * p.S + s] : p.fset[tile] + s * M * N;
    }

    // ---- K3: thread per packed bin k, both parity groups (outputs l0 + g + 2i), JH each.
    // The m loop is unrolled by JH so the sliding window rotates by register renaming (output i
    // at unrolled step u reads win[(i - u) mod JH]); loads run kPf steps ahead in registers.
    // Partition-group partials accumulate in the thread's own column of s_y (rows = outputs).
#ifndef TVOLAP_WIDE_KPF
#define TVOLAP_WIDE_KPF 2  // (diagnostic builds: _build.build_variant(..., ["TVOLAP_WIDE_KPF=4"]))
#endif
    constexpr int kPf = TVOLAP_WIDE_KPF;  // divides JH
    const float2* X[2];
    long bse[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        X[g] = p.xe + (s * 2 + ((l0 + g) & 1)) * p.T * N;
        bse[g] = ((l0 + g) >> 1) - p.tbase;  // t of output i = bse + i, of its partition-m input bse + i - m
    }
    // Packed bin 0 = (Re X_0, Re X_N) also needs the Nyquist products sum_m Im H . Im X (the hop
    // kernels' aux chain beside the complex one): warp 0 stages Im H[m][0] and Im X[g][t][0] in
    // shared memory and runs the Q x 2 x JH sequential fmaf chains, one per lane.
    float* s_auxh = reinterpret_cast<float*>(smem + lay.aux);
    float* s_auxx = s_auxh + M;                 // [2][M + JH]: t = bse - M + j
    float* s_auxr = s_auxx + 2 * (M + JH);      // [Q][2][JH]
    if (tid < 32) {
        for (int j = tid; j < M; j += 32) s_auxh[j] = __ldcg(H + (long)j * N).y;
        for (int j = tid; j < 2 * (M + JH); j += 32) {
            const int g = j >= M + JH, jj = j - g * (M + JH);
            s_auxx[j] = __ldcg((g ? X[1] + (bse[1] - M) * N : X[0] + (bse[0] - M) * N) + (long)jj * N).y;
        }
        __syncwarp();
        for (int c = tid; c < Q * 2 * JH; c += 32) {
            const int qq = c / (2 * JH), g = (c / JH) & 1, i = c % JH;
            const int mu0 = (int)((long)qq * M / Q), mu1 = (int)((long)(qq + 1) * M / Q);
            float aux = 0.f;
            for (int mm = mu0; mm < mu1; ++mm) aux = fmaf(s_auxh[mm], s_auxx[g * (M + JH) + M + i - mm], aux);
            s_auxr[c] = aux;
        }
        __syncwarp();
    }
    for (int k = tid; k < N; k += NT) {
        float2* col = s_y + k;  // this bin's outputs (rows jj), partition-group partials first
        for (int qq = 0; qq < Q; ++qq) {
            const int mu0 = (int)((long)qq * M / Q), mu1 = (int)((long)(qq + 1) * M / Q);
            float2 acc[2][JH];
            float2 win[2][JH];
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int i = 0; i < JH; ++i) {
                    acc[g][i] = make_float2(0.f, 0.f);
                    win[g][i] = __ldcg(X[g] + (bse[g] + i - mu0) * N + k);
                }
            // step m reads X[g][bse - m - 1] (the window's next entry) and H[m]; prefetches past
            // mu1 read padding (Xe front slots, pool tail rows) and are never used
            const float2* px0 = X[0] + (bse[0] - mu0 - 1) * N + k;
            const float2* px1 = X[1] + (bse[1] - mu0 - 1) * N + k;
            const float2* ph = H + (long)mu0 * N + k;
            float2 f0[kPf], f1[kPf], fh[kPf];
#pragma unroll
            for (int u = 0; u < kPf; ++u) {
                f0[u] = __ldcg(px0 - (long)u * N);
                f1[u] = __ldcg(px1 - (long)u * N);
                fh[u] = __ldcg(ph + (long)u * N);
            }
            px0 -= (long)kPf * N;
            px1 -= (long)kPf * N;
            ph += (long)kPf * N;
            auto step = [&](auto u_tag) {
                constexpr int u = decltype(u_tag)::value;
                constexpr int sl = u % kPf;
                const float2 x0 = f0[sl], x1 = f1[sl], h = fh[sl];
                f0[sl] = __ldcg(px0);
                f1[sl] = __ldcg(px1);
                fh[sl] = __ldcg(ph);
                px0 -= N;
                px1 -= N;
                ph += N;
#pragma unroll
                for (int g = 0; g < 2; ++g) {
#pragma unroll
                    for (int i = 0; i < JH; ++i) {
                        float2& a = acc[g][i];
                        const float2 x = win[g][(i - u) & (JH - 1)];
                        a.x = fmaf(h.x, x.x, a.x);
                        a.x = fmaf(-h.y, x.y, a.x);
                        a.y = fmaf(h.x, x.y, a.y);
                        a.y = fmaf(h.y, x.x, a.y);
                    }
                }
                win[0][(JH - 1 - u) & (JH - 1)] = x0;  // replaces the entry output JH-1 just used
                win[1][(JH - 1 - u) & (JH - 1)] = x1;
            };
            int m = mu0;
            for (; m + JH <= mu1; m += JH) {
                step(std::integral_constant<int, 0>{});
                step(std::integral_constant<int, 1>{});
                step(std::integral_constant<int, 2>{});
                step(std::integral_constant<int, 3>{});
                if constexpr (JH == 8) {
                    step(std::integral_constant<int, 4>{});
                    step(std::integral_constant<int, 5>{});
                    step(std::integral_constant<int, 6>{});
                    step(std::integral_constant<int, 7>{});
                }
            }
            const int rem = mu1 - m;  // < JH: the same unrolled steps, cut short
            if (rem > 0) step(std::integral_constant<int, 0>{});
            if (rem > 1) step(std::integral_constant<int, 1>{});
            if (rem > 2) step(std::integral_constant<int, 2>{});
            if constexpr (JH == 8) {
                if (rem > 3) step(std::integral_constant<int, 3>{});
                if (rem > 4) step(std::integral_constant<int, 4>{});
                if (rem > 5) step(std::integral_constant<int, 5>{});
                if (rem > 6) step(std::integral_constant<int, 6>{});
            }
            if (k == 0) {  // packed bin 0: two real products
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int i = 0; i < JH; ++i) {
                        const float a = s_auxr[(qq * 2 + g) * JH + i];
                        acc[g][i].x += a;
                        acc[g][i].y = a;
                    }
            }
#pragma unroll
            for (int g = 0; g < 2; ++g)
#pragma unroll
                for (int i = 0; i < JH; ++i) {
                    const int jj = g + 2 * i;
                    if (jj >= jt) continue;
                    float2* y = col + (size_t)jj * N;
                    if (qq == 0) {
                        *y = acc[g][i];
                    } else {
                        const float2 t = *y;
                        *y = make_float2(t.x + acc[g][i].x, t.y + acc[g][i].y);
                    }
                }
        }
    }
    __syncthreads();
    if (slot >= 0) {  // every read of the scratch set is done: drop its L2 lines unwritten, hand the slot on
        const char* sb = reinterpret_cast<const char*>(p.scratch + (size_t)slot * (M + kWideTail) * N);
        const size_t bytes = (size_t)M * N * sizeof(float2);
        for (size_t off = (size_t)tid * 128; off + 128 <= bytes; off += (size_t)NT * 128)
            asm volatile("discard.global.L2 [%0], 128;\n" ::"l"(sb + off) : "memory");
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            atomicExch(p.slot_lock + slot, 0u);
        }
    }

    // ---- K5: tangle + inverse FFT in batches of kWideFB frames, overlap-add per output sample
    constexpr int UPT = (L + 255) / 256;  // samples per thread (NT = 256)
    float st[UPT][3];
#pragma unroll
    for (int c = 0; c < UPT; ++c) st[c][0] = st[c][1] = st[c][2] = 0.f;
    const float sc = 1.0f / (float)N;
    float* head = p.thead + (s * p.ntiles + tile) * 6 * L;
    float* outp = p.out + s * p.out_stride + (long)l0r * L;
    // overlap-add of frames f0 .. f0 + nb - 1 whose time-domain samples (unscaled, 2N floats per
    // frame at stride fstride floats) start at ytd
    auto ola = [&](const float* ytd, size_t fstride, int f0, int nb) {
#pragma unroll
        for (int c = 0; c < UPT; ++c) {
            const int u = tid + c * 256;
            if (u >= L || tid >= NT) continue;
            for (int fi = 0; fi < nb; ++fi) {
                const int jj = f0 + fi;
                const float* yf = ytd + (size_t)fi * fstride + u;
                const float y0 = yf[0] * sc, y1 = yf[L] * sc, y2 = yf[2 * L] * sc, y3 = yf[3 * L] * sc;
                const float o = 0.5f * (y0 + st[c][0]);
                st[c][0] = st[c][1] + y1;
                st[c][1] = st[c][2] + y2;
                st[c][2] = y3;
                if (jj >= 3) {
                    outp[(long)jj * L + u] = o;
                } else if (jj == 0) {
                    head[0 * L + u] = y0;
                    head[1 * L + u] = y1;
                    head[2 * L + u] = y2;
                } else if (jj == 1) {
                    head[3 * L + u] = y0;
                    head[4 * L + u] = y1;
                } else {
                    head[5 * L + u] = y0;
                }
            }
        }
    };
    if (p.warp_fft && N >= 64 && N <= 1024) {  // 8 warp buffers of N = the two K5 buffers
        // one warp per frame, no CTA barriers: tangle into the warp's buffer (K5 buffers), then
        // the warp four-step inverse FFT writes the time-domain frame over its own Y row
        // (only this warp reads that row)
        const int warp = tid >> 5, lane = tid & 31;
        if constexpr (N >= 64 && N <= 512 && J == 16) {
            // two frames per warp in lockstep (rows 2w, 2w + 1 are contiguous), the tangle computed
            // in the transform's loads, results written over the two Y rows (in place)
            const int jj = 2 * warp;
            if (jj < jt) {
                float2* rows = s_y + (size_t)jj * N;
                auto ld = [&](int t, int n) { return tangle_packed(rows + (size_t)t * N, N, n, s_pk); };
                fft_warp4<true, N, false, 2, decltype(ld), true>(rows, p.tw + N, lane, ld);
            }
        } else {
            float2* wb = s_fa + (size_t)warp * N;
            for (int jj = warp; jj < jt; jj += NT >> 5) {
                float2* yrow = s_y + (size_t)jj * N;
                for (int kk = lane; kk < N; kk += 32) wb[kk] = tangle_packed(yrow, N, kk, s_pk);
                __syncwarp();
                if constexpr (N >= 64 && N <= 1024)
                    fft_warp4<true, N, false>(yrow, p.tw + N, lane, [&](int, int n) { return wb[n]; });
                __syncwarp();
            }
        }
        __syncthreads();
        ola(reinterpret_cast<const float*>(s_y), 2 * (size_t)N, 0, jt);
    } else {
        for (int f0 = 0; f0 < jt; f0 += kWideFB) {
            const int nb = min(kWideFB, jt - f0);
            for (int i = tid; i < nb * N; i += NT) {
                const int fi = i / N, kk = i - fi * N;
                s_fb[(size_t)fi * N + kk] = tangle_packed(s_y + (size_t)(f0 + fi) * N, N, kk, s_pk);
            }
            __syncthreads();
            ola(reinterpret_cast<const float*>(fft_batch<true, NC>(s_fb, s_fa, N, nb, s_tw, false, tid, NT)),
                2 * (size_t)N, f0, nb);
            __syncthreads();  // ytd / s_fb free for the next batch
        }
    }
    float* stt = p.tstate + (s * p.ntiles + tile) * 3 * L;
#pragma unroll
    for (int c = 0; c < UPT; ++c) {
        const int u = tid + c * 256;
        if (u >= L) continue;
        stt[u] = st[c][0];
        stt[L + u] = st[c][1];
        stt[2 * L + u] = st[c][2];
    }
}

// ============================================================================ period tiles
// K4 + K3 + K5 of one (lane, filter period) tile with the period's set transformed in partition
// groups into SHARED memory (C4: 2L = 1024 bins, M = 256, a fresh IR every 8 hops). A whole set
// (M x 2L complex = 2 MB for C4) per resident CTA does not stay in L2 (wide_mac_kernel's scratch
// slots: 148 x 2 MB), so here the tile walks its partitions in groups of G = NT / 32 (one warp per
// partition, 16 for C4): the group's IR taps (G x 2L contiguous floats, 64 KB) arrive by one
// cp.async.bulk (TMA) into a staging buffer signalled by an mbarrier — issued a whole group ahead,
// so the copy overlaps the previous group's MAC — each warp transforms its partition from the
// staging buffer into its spectra row (the warp four-step FFT + in-place untangle: the same
// operations as partition_warp_kernel), and the MAC reads the filter from shared memory:
//   Y_l += sum_{m in group} H[m] X_{l-2m}   (engine.cpp:85-92)
// A thread owns bins (t, t + NT) x both parities x JH outputs; the delay-line window slides by
// register renaming, X comes from Xe (L2) KPF steps ahead. The set's spectra never leave the SM.
// Then Y -> shared memory, tangle + inverse warp FFT one frame per warp, hop-2 overlap-add
// (engine.cpp:94-102), carries for wide_fixup_kernel — as in wide_mac_kernel.
// Partition sums run in m order inside each group and across groups (deterministic).
template <int NC>
struct PeriodLayout {
    static constexpr int N = NC, NT = NC / 2, G = NT / 32;
    static constexpr size_t a16c(size_t x) { return (x + 15) & ~size_t(15); }
    static constexpr size_t pk = 0;                                  // N + 2 pack phasors
    static constexpr size_t tw4 = a16c((size_t)(N + 2) * 8);        // N + 32 four-step twiddles
    static constexpr size_t spec = a16c(tw4 + (size_t)(N + 32) * 8);  // G spectra rows (Y, K5 buffers later)
    static constexpr size_t stage = spec + (size_t)G * N * 8;       // G x 2L IR taps
    static constexpr size_t auxx = stage + (size_t)G * N * 4;       // [2][G + 8] Im X[.][0]
    static constexpr size_t auxr = auxx + 2 * (G + 8) * 4;          // [16] running Nyquist sums
    static constexpr size_t bar = a16c(auxr + 16 * 4);
    static constexpr size_t total = bar + 16;
};

__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(bar), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
// one thread: bytes (multiple of 16, 16-byte aligned both ends) global -> shared, completion on bar
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // earlier generic accesses of dst are done
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}

#ifndef TVOLAP_PERIOD_KP
#define TVOLAP_PERIOD_KP 12  // period-tile MAC: X rows in flight per thread (JH + KP divides the group)
#endif

// f(integral_constant<int, u>) for u = 0 .. n - 1, fully unrolled
template <class F, int... us>
__device__ __forceinline__ void unroll_steps(F&& f, std::integer_sequence<int, us...>) {
    (f(std::integral_constant<int, us>{}), ...);
}

template <int NC, int JH>
__global__ void __launch_bounds__(NC / 2, 1) wide_period_kernel(const WideParams p) {
    using Lay = PeriodLayout<NC>;
    constexpr int N = NC, L = NC / 2, NT = Lay::NT, G = Lay::G, J = 2 * JH, KPF = 2;
    static_assert(J <= G && JH % KPF == 0 && G % JH == 0, "period tile geometry");
    extern __shared__ __align__(16) unsigned char smem[];
    float2* s_pk = reinterpret_cast<float2*>(smem + Lay::pk);
    float2* s_tw4 = reinterpret_cast<float2*>(smem + Lay::tw4);
    float2* s_spec = reinterpret_cast<float2*>(smem + Lay::spec);
    float* s_stage = reinterpret_cast<float*>(smem + Lay::stage);
    float* s_auxx = reinterpret_cast<float*>(smem + Lay::auxx);
    float* s_auxr = reinterpret_cast<float*>(smem + Lay::auxr);
    const unsigned bar = (unsigned)__cvta_generic_to_shared(smem + Lay::bar);
    const unsigned stage_sa = (unsigned)__cvta_generic_to_shared(s_stage);
    const unsigned spec_sa = (unsigned)__cvta_generic_to_shared(s_spec);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x;
    const long s = blockIdx.y;
    const int l0r = p.tile0[tile], jt = p.tile0[tile + 1] - l0r;
    const long l0 = p.hop0 + l0r;
    const int M = p.M;
    const int groups = M / G;
    // Tiles before the call's first switch use the engine's active set: its group spectra are
    // bulk-copied into the spectra rows instead of being transformed.
    const float* tir = p.tile_ir[tile];
    const float* h = tir ? tir + s * p.ir_len : nullptr;
    const float2* hset = tir ? nullptr : (p.fset_per_lane ? p.fset[(long)tile * p.S + s] : p.fset[tile] + s * M * N);
    // IR taps of group q: [q G N, (q + 1) G N) clipped to the IR; the rest of the staging row is zero
    auto group_bytes = [&](int q) -> unsigned {
        const long a = (long)q * G * N, b = min((long)(q + 1) * G * N, p.ir_len);
        return b > a ? (unsigned)((b - a) * 4) : 0u;
    };
    auto fetch = [&](int q) {  // one thread: the bytes group q needs, completion on bar
        if (h) {
            const unsigned nb = group_bytes(q);
            if (nb) bulk_g2s(stage_sa, h + (long)q * G * N, nb, bar);
            else mbar_arrive(bar);
        } else {
            bulk_g2s(spec_sa, hset + (size_t)q * G * N, (unsigned)(G * N * sizeof(float2)), bar);
        }
    };
    for (int i = tid; i <= N; i += NT) s_pk[i] = p.pk[i];
    for (int i = tid; i < N + 32; i += NT) s_tw4[i] = p.tw[N + i];
    if (tid < 16) s_auxr[tid] = 0.f;
    if (tid == 0) {
        mbar_init(bar, 1);
        fetch(0);
    }
    __syncthreads();

    const float2* X[2];
    long bse[2];
#pragma unroll
    for (int g = 0; g < 2; ++g) {
        X[g] = p.xe + (s * 2 + ((l0 + g) & 1)) * p.T * N;
        bse[g] = ((l0 + g) >> 1) - p.tbase;  // slot of output i at partition m: bse + i - m
    }
    float4 acc[2][JH];  // [parity g][output i]: bins 2 tid, 2 tid + 1
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int i = 0; i < JH; ++i) acc[g][i] = make_float4(0.f, 0.f, 0.f, 0.f);

    for (int q = 0; q < groups; ++q) {
        const int mu0 = q * G;
        mbar_wait(bar, (unsigned)(q & 1));
        if (h) {
            // ---- K4 of partitions mu0 .. mu0 + G - 1 (partition.cpp:20-51): warp w, partition
            // mu0 + w, from the staged taps; the warp four-step FFT + in-place untangle
            const float* src = s_stage + (size_t)warp * N;
            const long valid = (long)group_bytes(q) / 4 - (long)warp * N;  // taps of this partition staged
            float2* row = s_spec + (size_t)warp * N;
            if (valid >= N) {
                fft_warp4<false, N, true>(row, s_tw4, lane, [&](int, int n) -> float2 {
                    return *reinterpret_cast<const float2*>(src + 2 * n);
                });
            } else {
                fft_warp4<false, N, true>(row, s_tw4, lane, [&](int, int n) -> float2 {
                    const long i0 = 2 * n;
                    return make_float2(i0 < valid ? src[i0] : 0.f, i0 + 1 < valid ? src[i0 + 1] : 0.f);
                });
            }
            untangle_pairs_inplace_warp(row, N, s_pk, lane);
            __syncthreads();  // spectra of the group ready; staging consumed
            if (tid == 0 && q + 1 < groups) fetch(q + 1);  // overlaps this group's MAC
        }
        // Nyquist terms of packed bin 0 (warp 0): Im X[g][t][0] of the group's window into shared memory
        if (warp == 0) {
            for (int j = lane; j < 2 * (G + JH - 1); j += 32) {
                const int g = j >= G + JH - 1, jj = j - g * (G + JH - 1);  // slot bse - mu0 - (G - 1) + jj
                s_auxx[g * (G + 8) + jj] = __ldcg(X[g] + (bse[g] - mu0 - (G - 1) + jj) * N).y;
            }
        }
        // ---- K3 over the group (engine.cpp:85-92), filter rows from shared memory; a thread owns the
        // bin pair (2 tid, 2 tid + 1): one 16-byte load per operand row. The two parities run one
        // after the other (the filter rows are read twice from shared memory), so the window (JH
        // rows) and the loads in flight (KPF rows ahead) of one parity fit the register budget; the
        // m loop is unrolled by JH + KPF, one full turn of the window + prefetch registers, so the
        // rotation costs no moves.
        {
            constexpr int V = N / 2, KP = TVOLAP_PERIOD_KP < G - JH ? TVOLAP_PERIOD_KP : G - JH, U = JH + KP;  // float4 per row; prefetch depth; unroll
            static_assert(G % U == 0, "period tile: the group must hold whole unrolled turns");
            const float4* hrow = reinterpret_cast<const float4*>(s_spec) + tid;
            auto parity = [&](auto g_tag) {
                constexpr int g = decltype(g_tag)::value;
                const float4* xg = reinterpret_cast<const float4*>(X[g]) + tid;
                float4 win[JH], fx[KP];
#pragma unroll
                for (int i = 0; i < JH; ++i) win[i] = __ldcg(xg + (bse[g] + i - mu0) * V);
                // step m needs slot bse - m - 1 (the window's next entry); loads run KP steps ahead and
                // past the group read the next slots down (Xe front padding at the last group), unused
                const float4* px = xg + (bse[g] - mu0 - 1) * V;
#pragma unroll
                for (int k = 0; k < KP; ++k) fx[k] = __ldcg(px - (long)k * V);
                auto step = [&](auto u_tag, int mm) {
                    constexpr int u = decltype(u_tag)::value, sl = u % KP;
                    const float4 hv = hrow[(size_t)(mm + u) * V];
#pragma unroll
                    for (int i = 0; i < JH; ++i) {
                        float4& a = acc[g][i];
                        const float4 x = win[(i - u) & (JH - 1)];
                        a.x = fmaf(hv.x, x.x, a.x);
                        a.x = fmaf(-hv.y, x.y, a.x);
                        a.y = fmaf(hv.x, x.y, a.y);
                        a.y = fmaf(hv.y, x.x, a.y);
                        a.z = fmaf(hv.z, x.z, a.z);
                        a.z = fmaf(-hv.w, x.w, a.z);
                        a.w = fmaf(hv.z, x.w, a.w);
                        a.w = fmaf(hv.w, x.z, a.w);
                    }
                    win[(JH - 1 - u) & (JH - 1)] = fx[sl];
                    fx[sl] = __ldcg(px - (long)(mm + u + KP) * V);
                };
                for (int mm = 0; mm < G; mm += U)
                    unroll_steps([&](auto u_tag) { step(u_tag, mm); }, std::make_integer_sequence<int, U>{});
            };
            parity(std::integral_constant<int, 0>{});
            parity(std::integral_constant<int, 1>{});
        }
        if (warp == 0) {
            __syncwarp();
            if (lane < J) {  // output (g, i): sum_m Im H[m][0] Im X[g][bse + i - m][0], m in order
                const int g = lane / JH, i = lane % JH;
                float a = s_auxr[lane];
                for (int mm = 0; mm < G; ++mm)
                    a = fmaf(s_spec[(size_t)mm * N].y, s_auxx[g * (G + 8) + (G - 1) + i - mm], a);
                s_auxr[lane] = a;
            }
        }
        __syncthreads();  // every read of the group's spectra done
        if (!h && tid == 0 && q + 1 < groups) fetch(q + 1);  // copied spectra: the rows are free only now
    }

    // ---- Y rows jj = g + 2 i into shared memory (rows 0 .. J - 1), packed bin 0 fixed up
    float2* s_y = s_spec;
#pragma unroll
    for (int g = 0; g < 2; ++g)
#pragma unroll
        for (int i = 0; i < JH; ++i) {
            const int jj = g + 2 * i;
            float4 a = acc[g][i];
            if (tid == 0) {
                const float x = s_auxr[g * JH + i];
                a.x += x;
                a.y = x;
            }
            reinterpret_cast<float4*>(s_y + (size_t)jj * N)[tid] = a;
        }
    __syncthreads();
    // ---- K5: tangle + inverse warp FFT over the Y rows
    if constexpr (2 * J <= G) {  // one frame per warp, tangled into a warp buffer (rows J .. 2J - 1)
        for (int jj = warp; jj < jt; jj += NT / 32) {
            float2* yrow = s_y + (size_t)jj * N;
            float2* wb = s_y + (size_t)(J + (jj % J)) * N;
            for (int kk = lane; kk < N; kk += 32) wb[kk] = tangle_packed(yrow, N, kk, s_pk);
            __syncwarp();
            fft_warp4<true, N, false>(yrow, s_tw4, lane, [&](int, int n) { return wb[n]; });
            __syncwarp();
        }
    } else {  // no room for buffers: two frames per warp, tangled in the transform's loads, in place
        for (int jj = 2 * warp; jj < jt; jj += 2 * (NT / 32)) {  // rows jj, jj + 1 < J (J even)
            float2* rows = s_y + (size_t)jj * N;
            auto ld = [&](int t, int n) { return tangle_packed(rows + (size_t)t * N, N, n, s_pk); };
            fft_warp4<true, N, false, 2, decltype(ld), true>(rows, s_tw4, lane, ld);
        }
    }
    __syncthreads();
    const float sc = 1.0f / (float)N;
    float* head = p.thead + (s * p.ntiles + tile) * 6 * L;
    float* outp = p.out + s * p.out_stride + (long)l0r * L;
    const float* ytd = reinterpret_cast<const float*>(s_y);
    if (tid < L) {
        const int u = tid;
        float st0 = 0.f, st1 = 0.f, st2 = 0.f;
        for (int jj = 0; jj < jt; ++jj) {
            const float* yf = ytd + (size_t)jj * 2 * N + u;
            const float y0 = yf[0] * sc, y1 = yf[L] * sc, y2 = yf[2 * L] * sc, y3 = yf[3 * L] * sc;
            const float o = 0.5f * (y0 + st0);
            st0 = st1 + y1;
            st1 = st2 + y2;
            st2 = y3;
            if (jj >= 3) {
                outp[(long)jj * L + u] = o;
            } else if (jj == 0) {
                head[0 * L + u] = y0;
                head[1 * L + u] = y1;
                head[2 * L + u] = y2;
            } else if (jj == 1) {
                head[3 * L + u] = y0;
                head[4 * L + u] = y1;
            } else {
                head[5 * L + u] = y0;
            }
        }
        float* stt = p.tstate + (s * p.ntiles + tile) * 3 * L;
        stt[u] = st0;
        stt[L + u] = st1;
        stt[2 * L + u] = st2;
    }
}

// ============================================================================ bank pass
// K3 for bank engines with a per-hop schedule (C3, C5: every lane picks a bank entry every hop,
// so no filter spectrum is reused across the hops of a tile; engine.cpp:85-92 with the set
// exchanged before every hop, engine.hpp:55). One CTA per (tile, source x 32-float4 column
// chunk, partition group q). q is the SLOWEST grid axis: all resident CTAs read the same 1/Q
// slice of the bank, which stays L2-resident while the pass streams every (source, tile)
// through it, so the bank comes from HBM about once per pass instead of once per wave of CTAs.
// Thread = (column f, parity g, JO consecutive outputs of that parity) x E ears. Per partition
// step: one Xe load (L1-cached: the tile's other output groups re-read it a few steps later)
// and JO x E filter loads (L2 only), all issued KPF steps ahead into registers; the delay-line
// window slides by register renaming (m unrolled by JO). The partials of group q go to yq[q];
// bank_k5_kernel sums them in q order (deterministic).
template <int NC, int E, int JH, int JO, int KPF>
__global__ void __launch_bounds__(64 * (JH / JO), 512 / (64 * (JH / JO))) bank_mac_kernel(const WideParams p) {
    constexpr int N = NC, V4 = N / 2, CH = V4 / 32;
    static_assert(V4 % 32 == 0 && JH % JO == 0 && JO % KPF == 0 && (JO & (JO - 1)) == 0, "bank MAC geometry");
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int g = warp & 1, o = warp >> 1;
    const int s = blockIdx.y / CH, f = (blockIdx.y % CH) * 32 + lane;
    const int q = blockIdx.z;
    const int M = p.M, S = p.S;
    const int mq0 = (int)((long)q * M / p.Q), mq1 = (int)((long)(q + 1) * M / p.Q);
    // a CTA walks `tpc` consecutive tiles of its (source, partition group): the next tile's Xe
    // window is the previous one's shifted by JH slots, so most of its rows are still in L1
    const int tile_end = min(p.ntiles, ((int)blockIdx.x + 1) * p.tpc);
    for (int tile = (int)blockIdx.x * p.tpc; tile < tile_end; ++tile) {
    const int l0r = p.tile0[tile], jt = p.tile0[tile + 1] - l0r;
    if (g + 2 * o * JO >= jt) continue;  // a short tile: none of this warp's outputs exist (no barriers here)
    const long l0 = p.hop0 + l0r;
    const float4* pool4 = reinterpret_cast<const float4*>(p.pool);
    // filter rows of this thread's outputs (hop l0 + g + 2 (o JO + i)) at partition mq0
    const float4* hb[JO][E];
#pragma unroll
    for (int i = 0; i < JO; ++i) {
        const int jj = min(g + 2 * (o * JO + i), jt - 1);  // outputs past the tile: any valid entry, never stored
        const long ent = p.sched[(long)(l0r + jj) * S + s];
#pragma unroll
        for (int e = 0; e < E; ++e) hb[i][e] = pool4 + ((ent * E + e) * M + mq0) * V4 + f;
    }
    // Xe slot t of output i at step m: tb + i - m
    const float4* xs = reinterpret_cast<const float4*>(p.xe) + ((long)s * 2 + ((l0 + g) & 1)) * p.T * V4 + f;
    const long tb = ((l0 + g) >> 1) - p.tbase + o * JO;
    float4 acc[JO][E];
    float aux[JO][E];
    float4 win[JO];
#pragma unroll
    for (int i = 0; i < JO; ++i) {
        win[i] = __ldg(xs + (tb + i - mq0) * V4);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            acc[i][e] = make_float4(0.f, 0.f, 0.f, 0.f);
            aux[i][e] = 0.f;
        }
    }
    // step m needs X[tb - m - 1] (the window's next entry) and H_i[m]; loads run KPF steps ahead.
    // Prefetches past mq1 read the next entry's / the pool tail rows and the Xe front slots.
    const float4* px = xs + (tb - mq0 - 1) * V4;
    float4 fx[KPF], fh[KPF][JO][E];
#pragma unroll
    for (int k = 0; k < KPF; ++k) {
        fx[k] = __ldg(px - (long)k * V4);
#pragma unroll
        for (int i = 0; i < JO; ++i)
#pragma unroll
            for (int e = 0; e < E; ++e) fh[k][i][e] = __ldcg(hb[i][e] + (long)k * V4);
    }
    int m = mq0;
    auto step = [&](auto u_tag, auto guard_tag) {
        constexpr int u = decltype(u_tag)::value, sl = u % KPF;
        constexpr bool GUARD = decltype(guard_tag)::value;  // the group's last steps: no loads past mq1
        // FMAs on the operands loaded KPF steps ago, then the slot's registers take the loads of
        // step m + KPF (one register set per slot: no extra live copies)
#pragma unroll
        for (int i = 0; i < JO; ++i)
#pragma unroll
            for (int e = 0; e < E; ++e) cmac4(acc[i][e], aux[i][e], fh[sl][i][e], win[(i - u) & (JO - 1)]);
        win[(JO - 1 - u) & (JO - 1)] = fx[sl];  // replaces the entry output JO - 1 just used
        if (!GUARD || m + u + KPF < mq1) {
            fx[sl] = __ldg(px - (long)(u + KPF) * V4);
#pragma unroll
            for (int i = 0; i < JO; ++i)
#pragma unroll
                for (int e = 0; e < E; ++e) fh[sl][i][e] = __ldcg(hb[i][e] + (long)(u + KPF) * V4);
        }
    };
    auto advance = [&](int k) {
        px -= (long)k * V4;
#pragma unroll
        for (int i = 0; i < JO; ++i)
#pragma unroll
            for (int e = 0; e < E; ++e) hb[i][e] += (long)k * V4;
    };
    using IC0 = std::integral_constant<int, 0>;
    using IC1 = std::integral_constant<int, 1>;
    using IC2 = std::integral_constant<int, 2>;
    using IC3 = std::integral_constant<int, 3>;
    using IC4 = std::integral_constant<int, 4>;
    using IC5 = std::integral_constant<int, 5>;
    using IC6 = std::integral_constant<int, 6>;
    using IC7 = std::integral_constant<int, 7>;
    auto turn = [&](auto guard) {  // JO steps: one full turn of the register window
        step(IC0{}, guard);
        if constexpr (JO > 1) step(IC1{}, guard);
        if constexpr (JO > 2) {
            step(IC2{}, guard);
            step(IC3{}, guard);
        }
        if constexpr (JO > 4) {
            step(IC4{}, guard);
            step(IC5{}, guard);
            step(IC6{}, guard);
            step(IC7{}, guard);
        }
        advance(JO);
    };
    for (; m + JO + KPF <= mq1; m += JO) turn(std::false_type{});
    for (; m + JO <= mq1; m += JO) turn(std::true_type{});  // (the loads of the group's last KPF steps are skipped)
    const int rem = mq1 - m;  // < JO: the same unrolled steps, cut short
    if constexpr (JO > 1) {
        constexpr std::true_type G{};
        if (rem > 0) step(IC0{}, G);
        if constexpr (JO > 2) {
            if (rem > 1) step(IC1{}, G);
            if (rem > 2) step(IC2{}, G);
        }
        if constexpr (JO > 4) {
            if (rem > 3) step(IC3{}, G);
            if (rem > 4) step(IC4{}, G);
            if (rem > 5) step(IC5{}, G);
            if (rem > 6) step(IC6{}, G);
        }
    }
    float4* yq4 = reinterpret_cast<float4*>(p.yq);
#pragma unroll
    for (int i = 0; i < JO; ++i) {
        const int jj = g + 2 * (o * JO + i);
        if (jj >= jt) continue;
#pragma unroll
        for (int e = 0; e < E; ++e) {
            float4 a = acc[i][e];
            if (f == 0) {  // packed bin 0: two real products (Re X_0 H_0, Re X_N H_N)
                a.x += aux[i][e];
                a.y = aux[i][e];
            }
            __stcg(yq4 + ((((long)q * S + s) * E + e) * p.n + l0r + jj) * V4 + f, a);
        }
    }
    }  // tiles of this CTA
}

// K5 of the bank pass (spectral.cpp:127-158, engine.cpp:94-102): one CTA per (tile, output lane
// s * E + e): Y of the tile's hops = the partition-group partials summed in q order, tangle +
// inverse FFT (one warp per two frames, warp four-step, in place), then the overlap-add of the
// tile's outputs from its 4th hop on; the first three need the previous tile's carry
// (wide_fixup_kernel), exactly as in wide_mac_kernel.
template <int NC, int JH>
__global__ void __launch_bounds__(256) bank_k5_kernel(const WideParams p) {
    constexpr int N = NC, L = NC / 2, J = 2 * JH, V4 = N / 2;
    static_assert(N >= 64 && N <= 512, "bank K5 covers 64..512-point transforms");
    extern __shared__ __align__(16) unsigned char smem[];
    float2* s_pk = reinterpret_cast<float2*>(smem);
    float2* s_y = reinterpret_cast<float2*>(smem + a16((N + 2) * sizeof(float2)));
    const int tid = threadIdx.x, NT = 256, lane = tid & 31, warp = tid >> 5;
    const int tile = blockIdx.x;
    const long le = blockIdx.y;  // output lane s * E + e
    const long lanes = (long)p.S * p.E;
    const int l0r = p.tile0[tile], jt = p.tile0[tile + 1] - l0r;
    for (int i = tid; i <= N; i += NT) s_pk[i] = p.pk[i];
    const float4* yq4 = reinterpret_cast<const float4*>(p.yq);
    float4* y4 = reinterpret_cast<float4*>(s_y);
    for (int i = tid; i < J * V4; i += NT) {
        const int jj = i / V4, k4 = i - jj * V4;
        float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
        if (jj < jt) {
            const float4* src = yq4 + (le * p.n + l0r + jj) * V4 + k4;
            const long qs = lanes * p.n * V4;
            a = __ldcs(src);
            int q = 1;
            for (; q + 3 <= p.Q; q += 3) {  // three partials in flight, summed in q order
                const float4 b0 = __ldcs(src + (long)q * qs), b1 = __ldcs(src + (long)(q + 1) * qs),
                             b2 = __ldcs(src + (long)(q + 2) * qs);
                a = f4add(f4add(f4add(a, b0), b1), b2);
            }
            for (; q < p.Q; ++q) a = f4add(a, __ldcs(src + (long)q * qs));
        }
        y4[i] = a;
    }
    __syncthreads();
    for (int jj = 2 * warp; jj < jt; jj += 2 * (NT >> 5)) {  // rows jj, jj + 1 (J even: both exist)
        float2* rows = s_y + (size_t)jj * N;
        auto ld = [&](int t, int n) { return tangle_packed(rows + (size_t)t * N, N, n, s_pk); };
        fft_warp4<true, N, false, 2, decltype(ld), true>(rows, p.tw + N, lane, ld);
    }
    __syncthreads();
    const float sc = 1.0f / (float)N;
    float* head = p.thead + (le * p.ntiles + tile) * 6 * L;
    float* outp = p.out + le * p.out_stride + (long)l0r * L;
    const float* ytd = reinterpret_cast<const float*>(s_y);
    // hop-2 overlap-add (engine.cpp:94-102) without the serial carry: output jj needs only the
    // frames jj - 3 .. jj, summed in the carry's order ((y3 + y2) + y1, then y0) — the same
    // values the running carry gives (a tile has >= 3 hops)
    for (int idx = tid; idx < jt * L; idx += NT) {
        const int jj = idx / L, u = idx - jj * L;
        const float* yf = ytd + (size_t)jj * 2 * N + u;
        const float y0 = yf[0] * sc;
        if (jj >= 3) {
            const float y1 = yf[L - 2 * N] * sc, y2 = yf[2 * L - 4 * N] * sc, y3 = yf[3 * L - 6 * N] * sc;
            outp[(long)jj * L + u] = 0.5f * (y0 + ((y3 + y2) + y1));
        } else if (jj == 0) {
            head[0 * L + u] = y0;
            head[1 * L + u] = yf[L] * sc;
            head[2 * L + u] = yf[2 * L] * sc;
        } else if (jj == 1) {
            head[3 * L + u] = y0;
            head[4 * L + u] = yf[L] * sc;
        } else {
            head[5 * L + u] = y0;
        }
    }
    for (int u = tid; u < L; u += NT) {  // the carry after the tile's last hop
        const float* yl = ytd + (size_t)(jt - 1) * 2 * N + u;
        const float st2 = yl[3 * L] * sc;
        const float st1 = yl[3 * L - 2 * N] * sc + yl[2 * L] * sc;
        const float st0 = (yl[3 * L - 4 * N] * sc + yl[2 * L - 2 * N] * sc) + yl[L] * sc;
        float* stt = p.tstate + (le * p.ntiles + tile) * 3 * L;
        stt[u] = st0;
        stt[L + u] = st1;
        stt[2 * L + u] = st2;
    }
}

// First three outputs of every tile: the overlap-add recurrence of engine.cpp:97-102 continued
// from the carry after the previous tile (tile 0: the engine's carry from the previous call),
// in the order the sequential kernels evaluate it. Tile 0's threads also hand the last tile's
// carry and the last input hop (history) to the next call.
__global__ void wide_fixup_kernel(const WideParams p) {
    const int L = p.L;
    const long total = (long)p.S * p.E * p.ntiles * L;  // output lanes s * E + e
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long)gridDim.x * blockDim.x) {
        const int u = (int)(i % L);
        const int tile = (int)((i / L) % p.ntiles);
        const long s = i / ((long)L * p.ntiles);  // output lane
        const float* A = tile == 0 ? p.ola + s * 3 * L : p.tstate + (s * p.ntiles + tile - 1) * 3 * L;
        const float A0 = A[u], A1 = A[L + u], A2 = A[2 * L + u];
        const float* h = p.thead + (s * p.ntiles + tile) * 6 * L;
        const float o0 = 0.5f * (h[u] + A0);
        const float b0 = A1 + h[L + u];
        const float b1 = A2 + h[2 * L + u];
        const float o1 = 0.5f * (h[3 * L + u] + b0);
        const float c0 = b1 + h[4 * L + u];
        const float o2 = 0.5f * (h[5 * L + u] + c0);
        float* o = p.out + s * p.out_stride + (long)p.tile0[tile] * L + u;
        o[0] = o0;
        o[L] = o1;
        o[2 * L] = o2;
        if (tile == 0) {
            const float* last = p.tstate + (s * p.ntiles + p.ntiles - 1) * 3 * L;
            float* C = p.ola + s * 3 * L;
            C[u] = last[u];
            C[L + u] = last[L + u];
            C[2 * L + u] = last[2 * L + u];
            if (s % p.E == 0) {  // the source's last input hop (history), once per source
                const long src = s / p.E;
                p.hist[src * L + u] = p.in[src * p.in_stride + (long)(p.n - 1) * L + u];
            }
        }
    }
}

int sm_count() {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return sms;
}

int grid_cap(long work, int threads) {
    const long g = (work + threads - 1) / threads;
    return (int)std::max<long>(1, std::min<long>(g, (long)sm_count() * 16));
}

template <int NC>
cudaError_t launch_wide_t(const WideParams& p, int JH, cudaStream_t stream, cudaEvent_t t0, cudaEvent_t t1,
                          int parts) {
    cudaError_t err;
    if (parts & 1) {
        wide_head_kernel<<<grid_cap((long)p.S * 2 * (p.M + 2) * (NC / 2), 256), 256, 0, stream>>>(p);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if (p.warp_fft && NC == 64 && p.k1_small) {
            int per_sm = 0;
            if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wide_forward_small_kernel, 256, 0)) !=
                cudaSuccess)
                return err;
            const long items = (long)p.S * ((p.n + 31) / 32);
            const long grid = std::max<long>(1, std::min<long>(items, (long)sm_count() * std::max(1, per_sm)));
            wide_forward_small_kernel<<<(unsigned)grid, 256, 0, stream>>>(p);
            if ((err = cudaGetLastError()) != cudaSuccess) return err;
            return launch_wide_t<NC>(p, JH, stream, t0, t1, parts & ~1);
        }
        if (p.warp_fft && NC >= 64 && NC <= 1024) {
            const size_t smem = a16((NC + 2) * sizeof(float2)) + a16(NC * sizeof(float)) + 16 * (size_t)NC * sizeof(float2);
            if ((err = cudaFuncSetAttribute(wide_forward_warp_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            (int)smem)) != cudaSuccess)
                return err;
            int per_sm = 0;
            if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wide_forward_warp_kernel<NC>, 256, smem)) !=
                cudaSuccess)
                return err;
            const long pairs = ((long)p.S * p.n + 1) / 2;
            const long grid = std::max<long>(1, std::min<long>((pairs + 7) / 8, (long)sm_count() * std::max(1, per_sm)));
            wide_forward_warp_kernel<NC><<<(unsigned)grid, 256, smem, stream>>>(p);
            if ((err = cudaGetLastError()) != cudaSuccess) return err;
            return launch_wide_t<NC>(p, JH, stream, t0, t1, parts & ~1);
        }
        constexpr int F = kFwdF;
        const size_t smem = a16(NC * sizeof(float2)) + a16((NC + 2) * sizeof(float2)) + a16(NC * sizeof(float)) +
                            a16((F + 1) * (NC / 2) * sizeof(float)) + 2 * (size_t)F * NC * sizeof(float2);
        if ((err = cudaFuncSetAttribute(wide_forward_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)smem)) != cudaSuccess)
            return err;
        int per_sm = 0;
        if ((err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, wide_forward_kernel<NC>, 256, smem)) !=
            cudaSuccess)
            return err;
        const long items = (long)p.S * ((p.n + F - 1) / F);
        const long grid = std::max<long>(1, std::min<long>(items, (long)sm_count() * std::max(1, per_sm)));
        wide_forward_kernel<NC><<<(unsigned)grid, 256, smem, stream>>>(p);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
    if ((parts & 2) && p.period_smem) {
        if constexpr (NC == 512 || NC == 1024) {
            if (JH != 4 || !p.tile_ir) return cudaErrorInvalidValue;
            auto kern = wide_period_kernel<NC, 4>;
            constexpr size_t smem = PeriodLayout<NC>::total;
            if ((err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) !=
                cudaSuccess)
                return err;
            if (t0) cudaEventRecord(t0, stream);
            kern<<<dim3((unsigned)p.ntiles, (unsigned)p.S), NC / 2, smem, stream>>>(p);
            if ((err = cudaGetLastError()) != cudaSuccess) return err;
            if (t1) cudaEventRecord(t1, stream);
            wide_fixup_kernel<<<grid_cap((long)p.S * p.E * p.ntiles * p.L, 256), 256, 0, stream>>>(p);
            return cudaGetLastError();
        } else {
            return cudaErrorInvalidValue;
        }
    }
    if (parts & 2) {
        auto kern = JH == 8 ? wide_mac_kernel<NC, 8> : wide_mac_kernel<NC, 4>;
        const size_t smem = WideLayout(NC, 2 * JH, p.M, p.Q).total;
        if ((err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
            return err;
        if (t0) cudaEventRecord(t0, stream);
        kern<<<dim3((unsigned)p.ntiles, (unsigned)p.S), 256, smem, stream>>>(p);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
        if (t1) cudaEventRecord(t1, stream);
        wide_fixup_kernel<<<grid_cap((long)p.S * p.E * p.ntiles * p.L, 256), 256, 0, stream>>>(p);
        if ((err = cudaGetLastError()) != cudaSuccess) return err;
    }
    return cudaSuccess;
}

template <int NC, int E, int JH, int JO>
cudaError_t launch_bank_mac(const WideParams& p, cudaStream_t stream) {
    constexpr int KPF = 2;
    auto kern = bank_mac_kernel<NC, E, JH, JO, KPF>;
    const dim3 grid((unsigned)((p.ntiles + p.tpc - 1) / p.tpc), (unsigned)(p.S * (NC / 64)), (unsigned)p.Q);
    kern<<<grid, 64 * (JH / JO), 0, stream>>>(p);
    return cudaGetLastError();
}

template <int NC>
cudaError_t launch_bank_pass_t(const WideParams& p, int JH, cudaStream_t stream, cudaEvent_t t0, cudaEvent_t t1) {
    cudaError_t err = launch_wide_t<NC>(p, 8, stream, nullptr, nullptr, 1);  // head copy + K1 into Xe
    if (err != cudaSuccess) return err;
    if (t0) cudaEventRecord(t0, stream);
    if (p.E == 1 && JH == 32 && NC <= 128) err = launch_bank_mac<NC, 1, 32, 4>(p, stream);
    else if (p.E == 1 && JH == 16) err = launch_bank_mac<NC, 1, 16, 4>(p, stream);
    else if (p.E == 1 && JH == 8) err = launch_bank_mac<NC, 1, 8, 4>(p, stream);
    else if (p.E == 2 && JH == 8) err = launch_bank_mac<NC, 2, 8, 2>(p, stream);
    else if (p.E == 2 && JH == 16 && NC <= 256) err = launch_bank_mac<NC, 2, 16, 2>(p, stream);
    else return cudaErrorInvalidValue;
    if (err != cudaSuccess) return err;
    if (t1) cudaEventRecord(t1, stream);
    const size_t smem = a16((NC + 2) * sizeof(float2)) + (size_t)2 * JH * NC * sizeof(float2);
    auto k5 = JH == 16 ? bank_k5_kernel<NC, 16> : bank_k5_kernel<NC, 8>;
    if constexpr (NC <= 128)
        if (JH == 32) k5 = bank_k5_kernel<NC, 32>;
    if ((err = cudaFuncSetAttribute(k5, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)) != cudaSuccess)
        return err;
    k5<<<dim3((unsigned)p.ntiles, (unsigned)(p.S * p.E)), 256, smem, stream>>>(p);
    if ((err = cudaGetLastError()) != cudaSuccess) return err;
    wide_fixup_kernel<<<grid_cap((long)p.S * p.E * p.ntiles * p.L, 256), 256, 0, stream>>>(p);
    return cudaGetLastError();
}

template <int NC>
cudaError_t launch_partition_multi_t(int M, int S, long rows, const float* const* irs, long ir_len, float2* pool,
                                     const float2* tw, const float2* pk, cudaStream_t stream) {
    constexpr int kWarps = 8;
    const size_t smem = a16((NC + 2) * sizeof(float2)) + (size_t)kWarps * NC * sizeof(float2);
    cudaError_t err = cudaFuncSetAttribute(partition_multi_kernel<NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)smem);
    if (err != cudaSuccess) return err;
    int per_sm = 0;
    err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, partition_multi_kernel<NC>, 32 * kWarps, smem);
    if (err != cudaSuccess) return err;
    const long tasks = rows * M;
    const long grid = std::max<long>(1, std::min<long>((tasks + kWarps - 1) / kWarps,
                                                       (long)sm_count() * std::max(1, per_sm)));
    partition_multi_kernel<NC><<<(unsigned)grid, 32 * kWarps, smem, stream>>>(M, S, rows, irs, ir_len, pool, tw, pk);
    return cudaGetLastError();
}

}  // namespace

int wide_mac_ctas_per_sm(int L, int JH, int M, int Q) {
    const int N = 2 * L;
    const size_t smem = WideLayout(N, 2 * JH, M, Q).total;
    void (*fn)(const WideParams) = nullptr;
#define TVB_WK(n)                                                      \
    if (N == n) fn = JH == 8 ? wide_mac_kernel<n, 8> : wide_mac_kernel<n, 4>;
    TVB_WK(64) TVB_WK(128) TVB_WK(256) TVB_WK(512) TVB_WK(1024)
#undef TVB_WK
    if (!fn) return 0;
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem) != cudaSuccess) return 0;
    return per_sm;
}

bool period_kernel_supported(int L, int M, int JH, long ir_len) {
    const int N = 2 * L;
    return (N == 512 || N == 1024) && JH == 4 && M % (N / 64) == 0 && ir_len % 4 == 0;
}

bool wide_supported(int L) {
    const int N = 2 * L;
    return N == 64 || N == 128 || N == 256 || N == 512 || N == 1024;
}

size_t wide_mac_smem_bytes(int L, int JH, int M, int Q) { return WideLayout(2 * L, 2 * JH, M, Q).total; }

cudaError_t launch_wide(const WideParams& p, int JH, cudaStream_t stream, cudaEvent_t t0, cudaEvent_t t1, int parts) {
    switch (2 * p.L) {
        case 64: return launch_wide_t<64>(p, JH, stream, t0, t1, parts);
        case 128: return launch_wide_t<128>(p, JH, stream, t0, t1, parts);
        case 256: return launch_wide_t<256>(p, JH, stream, t0, t1, parts);
        case 512: return launch_wide_t<512>(p, JH, stream, t0, t1, parts);
        case 1024: return launch_wide_t<1024>(p, JH, stream, t0, t1, parts);
        default: return cudaErrorInvalidValue;
    }
}

bool bank_pass_supported(int L, int E, int JH) {
    const int N = 2 * L;
    if (!(N == 64 || N == 128 || N == 256 || N == 512)) return false;
    return (E == 1 && (JH == 16 || JH == 8 || (JH == 32 && N <= 128))) || (E == 2 && (JH == 8 || (JH == 16 && N <= 256)));
}

cudaError_t launch_bank_pass(const WideParams& p, int JH, cudaStream_t stream, cudaEvent_t t0, cudaEvent_t t1) {
    if (!bank_pass_supported(p.L, p.E, JH) || !p.warp_fft) return cudaErrorInvalidValue;
    switch (2 * p.L) {
        case 64: return launch_bank_pass_t<64>(p, JH, stream, t0, t1);
        case 128: return launch_bank_pass_t<128>(p, JH, stream, t0, t1);
        case 256: return launch_bank_pass_t<256>(p, JH, stream, t0, t1);
        case 512: return launch_bank_pass_t<512>(p, JH, stream, t0, t1);
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_partition_multi(int L, int M, int S, long rows, const float* const* irs, long ir_len, float2* pool,
                                   const float2* tw, const float2* pk, cudaStream_t stream) {
    switch (2 * L) {
        case 64: return launch_partition_multi_t<64>(M, S, rows, irs, ir_len, pool, tw, pk, stream);
        case 128: return launch_partition_multi_t<128>(M, S, rows, irs, ir_len, pool, tw, pk, stream);
        case 256: return launch_partition_multi_t<256>(M, S, rows, irs, ir_len, pool, tw, pk, stream);
        case 512: return launch_partition_multi_t<512>(M, S, rows, irs, ir_len, pool, tw, pk, stream);
        case 1024: return launch_partition_multi_t<1024>(M, S, rows, irs, ir_len, pool, tw, pk, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace tvb
