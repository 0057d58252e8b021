// Internal declarations shared by the kernel and host translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace tvb {

// Parameters of one launch of the fused per-hop kernel (K1+K2+K3+K5).
struct HopParams {
    int L;            // hop
    int M;            // partitions
    int D;            // delay-line slots per parity (>= M + hops per block / 2)
    int S;            // sources (input lanes)
    int P;            // CTAs per source (= cluster size)
    long hop0;        // global index of the first hop of this launch
    int n_hops;       // hops processed by this launch
    const float* in;  // in[s * in_stride + k * L + t]
    long in_stride;
    float* out;       // out[(s * E + e) * out_stride + k * L + t]
    long out_stride;
    float2* ring;          // frequency-domain delay line [S][2][D][2L] (packed bins)
    const float2* pool;    // filter spectra [entries][E][M][2L] (packed bins)
    const int* sched;      // bank entry per (hop, source) or per source; null -> entry_base + s
    long sched_stride;     // 0: same row for every hop
    int entry_base;
    float* hist;           // previous hop [S][L]
    float* ola;            // overlap-add accumulators [S][E][3L]
    const float2* tw;      // e^{-2 pi i t / 2L}, t < 2L
    const float2* pk;      // e^{-2 pi i k / 4L}, k <= 2L
    const float* win;      // periodic Hann, 2L
    // staged filter set transformed at the start of this launch (K4 fused), or new_ir == null
    const float* new_ir;   // new_ir[s * new_ir_stride + n], n < new_ir_len
    long new_ir_stride;
    long new_ir_len;
    float2* pool_w;        // writable view of pool
    int new_entry_base;    // pool entry of source 0 for the staged set
    int qm;                // one-hop kernel: partition groups (== the blocked kernel's, for bit-identical sums)
    // one-hop kernel, bank engines: the source of CTA cluster i is order[i] — sources sorted by
    // their selected bank entry, so the sources sharing an entry run side by side and its filter
    // rows come from HBM once per hop (L2 hits for the others); null = source i
    const int* order = nullptr;
    int ring_var = 0;      // one-hop bank launches on the bulk-copy ring kernel: geometry variant 1..4 (0: cluster hop kernel)
    // switching mode (tvolap_process_switching, hop-blocked set engines): a filter switch may
    // happen every sw_period hops of this launch; switch k (k < sw_count) installs the set
    // sw_irs[k] into pool entry sw_entry[k] (entry of source 0; -1: no switch at k).
    const float* const* sw_irs = nullptr;  // device array of sw_count device pointers
    const int* sw_entry = nullptr;         // device array of sw_count entries
    int sw_count = 0;
    int sw_period = 0;
    long sw_ir_stride = 0;                 // sw_irs[k][s * sw_ir_stride + n], n < sw_ir_len
    long sw_ir_len = 0;
};

// Process-wide launch knobs (tvolap_set_default_tuning): programmatic dependent launch of the hop
// kernels, warp-per-partition K4, its per-slice L2 prefetch.
extern long g_launch_pdl, g_launch_k4_warp, g_launch_k4_prefetch;

// Time-parallel pass (tvolap_wide.cu) over n hops of a device-resident call.
struct WideParams {
    int L, M, D, S, Q;     // Q: partition groups (the blocked kernel's, for bit-identical sums)
    long hop0;             // global index of the pass's first hop
    int n;                 // hops in the pass
    const float* in;       // in[s * in_stride + k * L + t], k < n
    long in_stride;
    float* out;            // out[s * out_stride + k * L + t]
    long out_stride;
    float2* ring;          // delay line [S][2][D][2L]: read before the pass, its last 2D hops written
    float2* xe;            // extended spectra [S][2][T][2L]: slot t of parity p = hop 2 (t + tbase) + p
    long T;
    long tbase;            // (hop0 >> 1) - M - kWideFront
    float* hist;           // [S][L]
    float* ola;            // [S][3L]
    const float2* tw;
    const float2* pk;
    const float* win;
    const float2* const* fset;  // per tile: filter set [S][M][2L]; fset_per_lane: per (tile, lane) [M][2L]
    int fset_per_lane;
    const int* tile0;           // tile k = hops tile0[k] .. tile0[k+1] of the pass (>= 3 hops each)
    int ntiles;
    float* tstate;              // overlap-add carry after each tile [S][ntiles][3][L]
    float* thead;               // first-three-output terms of each tile [S][ntiles][6][L]
    // fused K4 (one tile per period): tile_ir[tile] = the IR set in effect (null: use fset),
    // transformed by the tile into scratch slot [nslots][M + kWideTail][2L] (slot_lock: 0 = free)
    const float* const* tile_ir;
    long ir_len;
    float2* scratch;
    unsigned* slot_lock;
    int nslots;
    int stage_ir;               // fused K4: IR slices through a cp.async double buffer in shared memory
    int period_smem = 0;        // fused K4 in partition groups into shared memory (wide_period_kernel)
    int warp_fft;               // K1 / K5 with one warp per frame (warp four-step FFT) instead of the
                                // hop kernels' CTA Stockham (equal to fp32 rounding, not bit-identical)
    // bank pass (per-hop bank schedules, tvolap_wide.cu bank_mac_kernel / bank_k5_kernel)
    int E = 1;                  // ears: lanes s * E + e share source s's input spectra
    const float2* pool = nullptr;  // bank spectra [n_bank][E][M][2L]
    const int* sched = nullptr;    // bank entry of (pass hop h, source s): sched[h * S + s]
    float2* yq = nullptr;          // MAC partials per partition group [Q][S * E][n][2L]
    int tpc = 1;                   // bank MAC: consecutive tiles per CTA (L1 reuse of the Xe window)
    int k1_small = 1;              // 64-point K1 with 8 lanes per frame (wide_forward_small_kernel)
};
int wide_mac_ctas_per_sm(int L, int JH, int M, int Q);
bool wide_supported(int L);
// wide_period_kernel (fused K4 in shared-memory partition groups) covers this geometry
bool period_kernel_supported(int L, int M, int JH, long ir_len);
size_t wide_mac_smem_bytes(int L, int JH, int M, int Q);
constexpr int kWideFront = 8;   // Xe front padding slots per parity (tbase = (hop0 >> 1) - M - kWideFront)
constexpr int kWideTail = 8;    // spectra rows readable past the end of every filter set (prefetch)
// Bank pass: K1 as launch_wide part 1, then the per-hop-schedule MAC (tiles of 2 JH hops, JO
// outputs per thread, p.Q partition groups as the slowest grid axis), K5 + overlap-add per tile,
// fix-up. Events bracket the MAC launch.
cudaError_t launch_bank_pass(const WideParams& p, int JH, cudaStream_t stream, cudaEvent_t t0, cudaEvent_t t1);
bool bank_pass_supported(int L, int E, int JH);
// parts: 1 = head copy + forward FFTs, 2 = MAC/inverse tiles (+ fix-up); events bracket the tiles
cudaError_t launch_wide(const WideParams& p, int JH, cudaStream_t stream, cudaEvent_t t0, cudaEvent_t t1, int parts);
// K4 for rows = sets * S IRs: irs[row / S] + (row % S) * ir_len -> pool[(row * M + m) * 2L]
cudaError_t launch_partition_multi(int L, int M, int S, long rows, const float* const* irs, long ir_len, float2* pool,
                                   const float2* tw, const float2* pk, cudaStream_t stream);

size_t hop_kernel_smem_bytes(int L, int P, int E, int qm);
cudaError_t launch_hop_kernel(const HopParams& p, int E, int threads, cudaStream_t stream);
// persistent one-hop kernel with a cp.async.bulk ring (bank engines, P = 1): tvolap_kernels.cu
bool hop_ring_supported(const HopParams& p, int E, int threads);
cudaError_t launch_hop_ring_kernel(const HopParams& p, int E, int threads, cudaStream_t stream);

// Hop-blocked variant (2*JH hops per block, Q partition groups; threads == Q * (2L/P) when 2L/P < threads).
size_t block_kernel_smem_bytes(int L, int P, int E, int JH, bool bank, int threads);
cudaError_t launch_block_kernel(const HopParams& p, int E, int JH, int Q, int threads, cudaStream_t stream);

// K4: partition `rows` time-domain IRs (ir[row * ir_stride + n], n < ir_len) into
// M packed spectra each: pool[(row0 + row) * M + m][2L].
cudaError_t launch_partition(int L, int M, long rows, const float* ir, long ir_stride, long ir_len, float2* pool,
                             long row0, const float2* tw, const float2* pk, cudaStream_t stream,
                             bool pdl = false);

// Spectral primitives (tests of the reference's spectral.cpp contract).
cudaError_t launch_forward_real(long n, long batch, const float* x, float2* bins, const float2* tw,
                                const float2* pk, cudaStream_t stream);
cudaError_t launch_inverse_real(long n, long batch, const float2* bins, float* x, const float2* tw,
                                const float2* pk, cudaStream_t stream);
cudaError_t launch_mac(long nbins, long batch, const float2* acc, const float2* a, const float2* b, float2* out,
                       cudaStream_t stream);

// Workload generators (device twins of workload_host.cpp).
cudaError_t launch_gen_white(uint64_t seed, long lane0, long lanes, long t0, long n, float* out, long stride,
                             cudaStream_t stream);
cudaError_t launch_gen_irs(uint64_t seed, long count, const long* lanes, const long* ears, const long* ks,
                           const double* t60, double fs, long len, float* out, cudaStream_t stream);
cudaError_t launch_mix(long sources, long ears, long samples, const float* out, long out_stride, float* mix,
                       long mix_stride, cudaStream_t stream);
// peer-memory mix: per-GPU source sums stored into slot `rank` of every rank's gather buffer
// (slots[r] = rank r's buffer [world][ears][cap]), then the rank-ordered sum of the slots
cudaError_t launch_mix_scatter(long sources, long ears, long samples, const float* out, long out_stride,
                               float* const* slots, int world, int rank, long cap, cudaStream_t stream);
cudaError_t launch_mix_gather(long ears, long samples, const float* gather, int world, long cap, float* mix,
                              long mix_stride, cudaStream_t stream);

// comparison convolvers: OLA / OLS / WOLA block FFT convolution (kind 2/3/4)
// and the direct-form FIR of "tdc" / "cf-tdc"
cudaError_t launch_fbconv(int kind, int B, long channels, long n_hops, const float* in, long in_stride, float* prev,
                          const float2* spec, const float* win, const float2* tw, const float2* pk, float* yhat,
                          float* out, long out_stride, float* rem, cudaStream_t stream);
cudaError_t launch_fir(int taps, long channels, long T, const float* xx, long xx_stride, const float* h,
                       const float* h_old, float* out, long out_stride, long fade_len, long fade_elapsed0,
                       long fade_duration, int fade_shape, cudaStream_t stream);

}  // namespace tvb
