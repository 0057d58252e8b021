// Host side of the B200 TVOLAP engine: the C-ABI of include/tvolap_b200.h.
//
// Mirrors tvolap::TvolapEngine / TvolapProcessor (proj/include/tvolap/engine.hpp:33-94,
// proj/src/engine.cpp:9-118, proj/src/reference.cpp:328-342): construction
// partitions the IRs on the device, process() runs the one-hop kernel,
// process_hops() the hop-blocked kernel, exchange_filter() stages a replacement
// set that is latched at the next hop boundary (last staged wins, a staged set
// survives reset). Device state:
//   ring  [S][2][D][2L] complex64  frequency-domain delay line, D = M + 8 slots per parity
//   pool  [entries][E][M][2L]       filter partition spectra; set engines keep
//                                   three slots of S entries (active / staged / spare),
//                                   bank engines the whole bank
//   hist  [S][L], ola [S][E][3L]    per-lane time-domain state
// Host pointers are streamed through pinned staging buffers: H2D, kernel and
// D2H of consecutive chunks run on three streams so copies overlap compute.
// Staged filter sets are transformed (K4) on a high-priority side stream.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/tvolap_b200.h"
#include "tvolap_fft.cuh"
#include "tvolap_internal.cuh"

using tvb::HopParams;

namespace {

thread_local std::string g_err;

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

struct CudaFail {
    cudaError_t err;
    const char* what;
};

#define CK(expr)                                                     \
    do {                                                             \
        cudaError_t e_ = (expr);                                     \
        if (e_ != cudaSuccess) throw CudaFail{e_, #expr};            \
    } while (0)

struct ApiError {
    int code;
    std::string msg;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return TVOLAP_OK;
    } catch (const ApiError& e) {
        return set_err(e.code, e.msg);
    } catch (const CudaFail& e) {
        return set_err(TVOLAP_ERR_CUDA, std::string("CUDA error ") + cudaGetErrorName(e.err) + " (" +
                                            cudaGetErrorString(e.err) + ") in " + e.what);
    } catch (const std::exception& e) {
        return set_err(TVOLAP_ERR_CUDA, e.what());
    }
}

bool is_pow2(long n) { return n > 0 && (n & (n - 1)) == 0; }

enum class Mem { Device, Pinned, Pageable };

Mem classify(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return Mem::Pageable;
    }
    switch (a.type) {
        case cudaMemoryTypeDevice:
        case cudaMemoryTypeManaged:
            return Mem::Device;
        case cudaMemoryTypeHost:
            return Mem::Pinned;
        default:
            return Mem::Pageable;
    }
}

void require_device(int device) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        throw ApiError{TVOLAP_ERR_CUDA, "no CUDA device: the B200 engine has no CPU fallback"};
    }
    if (device < 0 || device >= n) throw ApiError{TVOLAP_ERR_CUDA, "device index out of range"};
    CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        throw ApiError{TVOLAP_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100 (Blackwell)"};
}

// fp64 tables rounded once to fp32 (spectral.cpp:50-61 formulas).
struct Tables {
    std::vector<float2> tw, pk;
    explicit Tables(long nc) {
        const double pi = 3.14159265358979323846264338327950288;
        // [stage table (nc) | warp four-step tables (nc + 32)]
        auto mk = [](double c, double s) { return make_float2((float)c, (float)s); };
        tw.assign(2 * nc + 32, make_float2(0.f, 0.f));
        tvb::fft_stage_twiddles((int)nc, tw.data(), mk);
        if (nc >= 64 && nc <= 1024) tvb::fft_warp_twiddles((int)nc, tw.data() + nc, mk);
        pk.resize(nc + 2);
        for (long k = 0; k <= nc; ++k) {
            const double a = -2.0 * pi * (double)k / (double)(2 * nc);
            pk[k] = make_float2((float)std::cos(a), (float)std::sin(a));
        }
        pk[nc + 1] = make_float2(0.f, 0.f);
    }
};

std::vector<float> hann(long hop) {  // partition.cpp:10-18
    const double pi = 3.14159265358979323846264338327950288;
    std::vector<float> w(2 * hop);
    for (long i = 0; i < 2 * hop; ++i) w[i] = (float)(1.0 - std::cos(2.0 * pi * (double)i / (double)(2 * hop)));
    return w;
}

template <class T>
T* dalloc(size_t count) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    return static_cast<T*>(p);
}

constexpr int kMaxJH = 8;  // largest hop block / 2 (ring slack per parity)
// Filter-set slots: active + staged + one more, so the transform of the next staged set
// may start while the two previous periods' hop kernels still read their sets.
constexpr int kSlots = 3;
// Host-IR upload buffers: uploads run on their own stream up to this many sets ahead.
constexpr int kIrStage = 4;


}  // namespace

// A device-resident FilterPartitionSet (partition.hpp:21-32): S x M packed partition spectra,
// computed once by K4 and immutable afterwards; shared by reference count (the engines that
// hold it as their active or staged filter keep it alive), like the reference's
// shared_ptr<const FilterPartitionSet>.
struct tvolap_set {
    int device = 0;
    long L = 0, M = 0, S = 0, N = 0, source_length = 0;
    float2* spec = nullptr;  // [S][M][2L] (+ kWideTail rows)
    std::atomic<int> refs{1};
};

namespace {
void set_retain(const tvolap_set* s) {
    if (s) const_cast<tvolap_set*>(s)->refs.fetch_add(1);
}
void set_release(const tvolap_set* cs) {
    auto* s = const_cast<tvolap_set*>(cs);
    if (!s || s->refs.fetch_sub(1) != 1) return;
    cudaSetDevice(s->device);
    cudaFree(s->spec);  // implicitly waits for the device work that may still read it
    delete s;
}
}  // namespace

struct tvolap_engine {
    int device = 0;
    int sms = 148;                   // SM count of the device (queried at creation)
    long L = 0, M = 0, S = 0, E = 1, N = 0;
    bool bank = false;
    long n_bank = 0;
    cudaStream_t own = nullptr, stream = nullptr, side = nullptr, h2d = nullptr, d2h = nullptr, upl = nullptr;
    cudaEvent_t ev_side = nullptr, ev_main = nullptr, ev_start = nullptr;
    cudaEvent_t ev_slot[kSlots] = {};  // last hop kernel that read each filter slot
    float2 *ring = nullptr, *pool = nullptr, *tw = nullptr, *pk = nullptr;
    // filter held as an external device set (tvolap_create_from_set / tvolap_exchange_set): read in
    // place, no K4; null = the pool slot `active`
    const tvolap_set* active_ext = nullptr;
    const tvolap_set* pending_ext = nullptr;
    float *win = nullptr, *hist = nullptr, *ola = nullptr;
    int* d_sel = nullptr;            // [S] latched selection | [S] sources sorted by it (d_sel + S)
    std::vector<int> sel, staged;
    int* h_sel[2] = {};              // pinned host staging of d_sel's two halves (alternating;
    cudaEvent_t ev_sel[2] = {};      // a pageable 32 KB upload costs ~25 us per hop, pinned ~7)
    int sel_next = 0;
    bool sel_dirty = false;          // `sel` not yet uploaded: done right before the next hop launch,
                                     // after the call's input copy is queued (host sort off the path)
    bool order_valid = false;        // d_sel + S holds the order of the current selection
    long entry_order = 1;            // "entry_order": one-hop kernel visits sources grouped by entry
    bool sel_staged = false;
    int active = 0;
    bool pending = false;
    float* d_irstage = nullptr;
    size_t irstage_cap = 0;
    // staged replacement set, transformed by the first kernel of the next process call
    const float* staged_ir = nullptr;
    long staged_len = 0;
    int staged_buf = -1;             // upload buffer holding it (-1: caller's device memory)
    float* d_irst[kIrStage] = {};    // host-IR upload buffers (round robin)
    size_t irst_cap[kIrStage] = {};
    int irst_next = 0;
    long ir_stages = 1;              // upload buffers in use (<= kIrStage); 1 measured best: uploads
                                     // running ahead delay the audio H2D on the critical path
    cudaEvent_t ev_up[kIrStage] = {}, ev_used[kIrStage] = {};  // upload landed / consuming kernel done
    const float* launch_new_ir = nullptr;  // latched: the next launch transforms this set
    long launch_new_len = 0;
    int launch_buf = -1;
    long k4_side = 1;                // 1: transform staged sets on the side stream (overlapping hops)
    bool staged_on_side = false;     // the pending set was transformed on the side stream
    long k4_stream = 1;              // 1: transform at latch time on the engine stream (PDL chain)
    // switching launches (tvolap_process_switching): per-switch IR pointers / pool entries
    const float** d_sw_irs = nullptr;
    int* d_sw_entry = nullptr;
    long sw_cap = 0;
    const float* const* sw_irs_launch = nullptr;  // set only around a switching launch
    const int* sw_entry_launch = nullptr;
    int sw_count_launch = 0, sw_period_launch = 0;
    long sw_len_launch = 0;
    // pinned-host switching pipeline: double-buffered device staging of hops, sets and outputs
    float *swh_x[2] = {}, *swh_y[2] = {}, *swh_ir[2] = {};
    long swh_cap_x = 0, swh_cap_ir = 0;
    bool staged_in_stream = false;   // the pending set is transformed by latch() on the engine stream
    // time-parallel pass (tvolap_wide.cu): extended spectra, the call's filter sets, tile tables
    float2 *wide_xe = nullptr, *wide_pool = nullptr;
    float *wide_state = nullptr, *wide_head = nullptr;
    const float2** d_wide_fset = nullptr;
    const float** d_wide_irs = nullptr;
    int* d_wide_tile0 = nullptr;
    size_t wide_xe_cap = 0, wide_pool_cap = 0, wide_tile_cap = 0, wide_fset_cap = 0, wide_sw_cap = 0;
    size_t wide_state_cap = 0, wide_head_cap = 0;
    float2* wide_scratch = nullptr;      // fused K4: one set per resident MAC CTA
    unsigned* wide_lock = nullptr;
    const float** d_wide_tile_ir = nullptr;
    size_t wide_scratch_cap = 0, wide_lock_cap = 0, wide_tile_ir_cap = 0;
    long wide_mode = 1;              // "wide": 0 off, 1 auto, 2 whenever supported
    // bank pass (per-hop bank schedules on device-resident hops): MAC partials per partition group
    float2* bank_yq = nullptr;
    size_t bank_yq_cap = 0;
    long bank_pass = 1;              // 0: per-hop schedules stay on the hop-blocked kernel
    long bank_pass_mb = 32768;       // Xe + partials budget per pass
    long bank_pass_hops = 0;         // max hops per pass (0: by the budget)
    long bank_pass_tpc = 0;          // bank MAC tiles per CTA (0: all tiles of the pass)
    long zero_copy = 1;              // one-hop calls on pinned host buffers: the kernel reads / writes them in place
    long hop_ring = 0;               // one-hop calls of bank engines on the persistent bulk-copy ring kernel
                                     // (geometry variant 1..4; measured no faster: profiles/r02_ab_hop_ring.txt)
    long k1_small = 1;               // 64-point K1 of the passes with 8 lanes per frame
    long bank_pass_jh = 0;           // half the hops of a bank-pass tile (0: auto; 8, 16 or 32)
    long bank_pass_q = 0;            // partition groups of the bank pass (0: auto, bank slice <= 40 MB)
    uint64_t wide_passes = 0;
    uint64_t ring_launches = 0;   // one-hop launches on the bulk-copy ring kernel
    long pipe_merge = 1;             // "pipe_merge": one H2D copy per run of host-contiguous sets
    long wide_warp_fft = 1;          // "wide_warp_fft": 1 warp FFTs for K1/K5 (0: bit-identical Stockham)
    // further tuning knobs (tvolap_set_tuning; defaults = the measured-best choices)
    long wide_q = -1;                // wide pass partition groups (-1: auto)
    long wide_stage = 1;             // fused K4 IR slices through a cp.async double buffer
    long wide_pool_mb = 8192;        // unfused wide pass: filter-set pool budget
    long wide_fuse = 1;              // fused K4 in the wide MAC tiles
    long wide_xe_mb = 4096;          // wide pass: extended-spectra budget
    long wide_period = 1;            // fused K4 in shared-memory partition groups (wide_period_kernel)
    long k4_gap_mult = 1;            // switching launch: K4 units per barrier gap (x warps x CTAs)
    long sw_1024 = 0;                // switching launch also for 1024-point transforms
    long pipe_mb = 64;               // pinned switching pipeline chunk
    long pipe_log2 = 25;             // pinned hop pipeline chunk (floats, log2)
    long fix_p = 0, fix_nt = 0, fix_pb = 0, fix_jh = 0, ntb = 256;  // geometry overrides (0: auto)
    // chunked host pipeline
    long chunk_hops = 0, host_chunk = 0;
    float *d_in[2] = {}, *d_out[2] = {}, *h_in[2] = {}, *h_out[2] = {};
    int* d_sch[2] = {};
    long sch_cap = 0;
    cudaEvent_t ev_in[2] = {}, ev_k[2] = {}, ev_o[2] = {};
    bool profiling = false;  // bracket every hop-kernel launch with CUDA events
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_events;
    size_t prof_used = 0;
    long chunk_seq = 0;     // alternates the double-buffered staging across calls
    bool host_async = false;  // pinned host I/O returns before completion
    int P = 1, NT = 256;           // streaming (one hop at a time) kernel
    int JH = 4, QB = 1, NTB = 256;   // hop-blocked kernel: 2*JH hops per block, QB partition groups
    int PB = 1;                      // hop-blocked kernel: CTAs (cluster size) per source
    int QM = 1;                      // partition groups of both kernels (bit-identical sums)
    bool geometry_fixed = false;     // set by tvolap_set_launch_config / set_block_config / tuning
    long D = 0;                      // delay-line slots per parity (M + kMaxJH)
    long block_min = 4;              // process_hops calls with >= block_min hops use the blocked kernel
    uint64_t fwd = 0, inv = 0, macs = 0, launches = 0;
    long hops = 0;
    std::mutex mu;

    ~tvolap_engine() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        if (side) cudaStreamSynchronize(side);
        set_release(active_ext);
        set_release(pending_ext);
        for (void* p : {(void*)ring, (void*)pool, (void*)tw, (void*)pk, (void*)win, (void*)hist, (void*)ola,
                        (void*)d_sel, (void*)d_irstage, (void*)d_irst[0], (void*)d_irst[1], (void*)d_irst[2],
                        (void*)d_irst[3], (void*)d_in[0],
                        (void*)d_in[1], (void*)d_out[0],
                        (void*)d_out[1], (void*)d_sch[0], (void*)d_sch[1], (void*)d_sw_irs, (void*)d_sw_entry,
                        (void*)swh_x[0], (void*)swh_x[1], (void*)swh_y[0], (void*)swh_y[1], (void*)swh_ir[0],
                        (void*)swh_ir[1], (void*)wide_xe, (void*)wide_pool, (void*)wide_state, (void*)wide_head,
                        (void*)d_wide_fset, (void*)d_wide_irs, (void*)d_wide_tile0, (void*)wide_scratch,
                        (void*)wide_lock, (void*)d_wide_tile_ir, (void*)bank_yq})
            if (p) cudaFree(p);
        for (float* p : {h_in[0], h_in[1], h_out[0], h_out[1]})
            if (p) cudaFreeHost(p);
        for (int* p : {h_sel[0], h_sel[1]})
            if (p) cudaFreeHost(p);
        for (cudaEvent_t ev : {ev_side, ev_main, ev_start, ev_in[0], ev_in[1], ev_k[0], ev_k[1], ev_o[0], ev_o[1],
                                ev_slot[0], ev_slot[1], ev_slot[2], ev_up[0], ev_up[1], ev_up[2], ev_up[3],
                                ev_used[0], ev_used[1], ev_used[2], ev_used[3], ev_sel[0], ev_sel[1]})
            if (ev) cudaEventDestroy(ev);
        for (auto& pr : prof_events) {
            cudaEventDestroy(pr.first);
            cudaEventDestroy(pr.second);
        }
        for (cudaStream_t s : {own, side, h2d, d2h, upl})
            if (s) cudaStreamDestroy(s);
    }
};

namespace {

void pick_launch_config(tvolap_engine* e) {
    // P: CTAs per source. Enough CTAs to cover the 148 SMs, never a slice
    // smaller than one float4 per thread group.
    long p = 1;
    while (p < 8 && p * 2 <= e->L && e->S * p < e->sms) p *= 2;
    e->P = (int)p;
    e->NT = 256;
    if (e->fix_p > 0) e->P = (int)e->fix_p;
    if (e->fix_nt > 0) e->NT = (int)e->fix_nt;
    // (same-box A/B, C2 exchange every 16 hops: K4 on a side stream 2.82 us/hop, + PDL 2.77,
    // in-stream K4 chained by PDL 2.53, profiles/r01_ab_pdl.txt: k4_side = k4_stream = 1)
}

// Blocked kernel geometry for the current P: W = 2L/P (parity x float4) work items per CTA.
void pick_block_geometry(tvolap_engine* e) {
    // Heuristic from the launch sweep (scripts/sweep_launch.py, profiles/): filter-set engines
    // want ~128+ CTAs and the longest block that fits; long hops want the largest cluster (the
    // per-CTA spectrum slice shrinks, two CTAs fit per SM); bank engines one CTA per source.
    if (!e->geometry_fixed) {
        long pb = 1;
        const long cap = std::min<long>(8, e->L);
        if (e->bank) {
            while (pb < cap && e->S * pb < 256) pb *= 2;
            // sweep: C5 (one ear) 16-hop blocks 118 us/hop vs 158 (8) vs 292 (one-hop kernel);
            // C3 (two ears) cluster of 2 with 8-hop blocks 60 us/hop vs 65 (P1, J4)
            e->JH = e->E == 2 ? 4 : 8;
            if (e->E == 2) pb = std::min<long>(cap, std::max<long>(pb, 2));
        } else {
            // sweep (profiles/r01_sweep_j16.jsonl): 16-hop blocks with the float2 unified MAC win
            // everywhere they fit — C2 1.60 vs 2.34 us/hop (8-hop), C1 0.83 vs 1.21, C4 (P = 8)
            // 31.6 vs 42.2; the shared-memory check below halves JH where they do not fit.
            while (pb < cap && e->S * pb < 256) pb *= 2;
            if (e->L >= 512) pb = cap;
            e->JH = 8;
        }
        e->PB = (int)pb;
        if (e->fix_pb > 0) e->PB = (int)e->fix_pb;
        if (e->fix_jh > 0) e->JH = (int)e->fix_jh;
    }
    const long W = e->N / e->PB;
    e->NTB = (int)std::max<long>(32, std::min<long>(256, e->ntb));  // A/B knob; 256 measured best
    e->QB = 1;
    if (W < e->NTB) {
        e->QB = (int)(e->NTB / W);
        while (e->QB > e->M && e->QB > 1) {
            e->QB /= 2;
            e->NTB /= 2;
        }
    }
    if (e->NTB < 32) e->NTB = 32, e->QB = (int)std::max<long>(1, 32 / W);
    while (e->JH > 1 && tvb::block_kernel_smem_bytes((int)e->L, e->PB, (int)e->E, e->JH, e->bank, e->NTB) > 227 * 1024)
        e->JH /= 2;
    // The blocked kernel splits the partitions into NTB / (items per group) contiguous groups;
    // the one-hop kernel uses the same grouping so process() and process_hops() agree bit for bit.
    const long Vb = e->N / (2 * e->PB);
    const long items = (!e->bank && e->JH <= 4) ? Vb : 2 * Vb;  // float4 unified vs float2 unified / per-parity
    e->QM = items < e->NTB ? (int)(e->NTB / items) : 1;
}

// Threads of the opt-in ring variant: one per (partition group, float4 column), as its stages assume.
int hop_ring_threads(const tvolap_engine* e) {
    const long t = std::min<long>(1024, e->QM * (e->N / (2 * e->P)));
    return (int)std::max<long>(32, (t + 31) / 32 * 32);
}

// Threads of the one-hop kernel: QM partition groups x the slice's float4 columns.
int hop_threads(const tvolap_engine* e) {
    // tuning nt: fewer threads than QM x V make each MAC thread stride over several columns of its
    // group (same groups, same summation order: bit-identical), trading warps for resident CTAs
    if (e->fix_nt >= 32) return (int)e->fix_nt;
    const long V = e->N / (2 * e->P);
    long t = std::min<long>(1024, e->QM * V);
    t = std::max<long>(32, (t + 31) / 32 * 32);
    // bank engines with a slice one warp wide (C5: V = 32, 8 groups): two-warp CTAs, each MAC
    // thread walking 4 columns — 16 resident CTAs per SM instead of 4, cheaper barriers around
    // the 64-point transforms (C5 hop kernel 246.5 -> 240.5 us, profiles/r02_ab_hop_threads.txt)
    if (e->bank && e->P == 1 && V <= 32 && t > 64) t = 64;
    return (int)t;
}

void validate_launch(const tvolap_engine* e, int P, int NT) {
    if (P < 1 || P > 8 || !is_pow2(P) || P > e->L)
        throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "cluster size P must be 1, 2, 4 or 8 and <= L"};
    if (NT < 32 || NT > 1024 || !is_pow2(NT))
        throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "threads per CTA must be a power of two in [32, 1024]"};
    const size_t smem = tvb::hop_kernel_smem_bytes((int)e->L, P, (int)e->E, std::max(1, e->QM));
    (void)NT;
    if (smem > 227 * 1024)
        throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION,
                       "hop L=" + std::to_string(e->L) + " needs " + std::to_string(smem) +
                           " B of shared memory per CTA (max 227 KB)"};
}

void apply_default_tuning(tvolap_engine* e);

void init_common(tvolap_engine* e, int device, long hop, long sources, long ears, long partitions) {
    e->device = device;
    CK(cudaDeviceGetAttribute(&e->sms, cudaDevAttrMultiProcessorCount, device));
    e->L = hop;
    e->N = 2 * hop;
    e->S = sources;
    e->E = ears;
    e->M = partitions;
    e->D = partitions + kMaxJH;
    CK(cudaStreamCreateWithFlags(&e->own, cudaStreamNonBlocking));
    int prio_lo = 0, prio_hi = 0;
    CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    // staged-filter transforms sit on the critical path of the next hop: schedule them first
    CK(cudaStreamCreateWithPriority(&e->side, cudaStreamNonBlocking, prio_hi));
    CK(cudaStreamCreateWithFlags(&e->h2d, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&e->d2h, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&e->upl, cudaStreamNonBlocking));
    e->stream = e->own;
    for (cudaEvent_t* ev : {&e->ev_side, &e->ev_main, &e->ev_start, &e->ev_in[0], &e->ev_in[1], &e->ev_k[0],
                            &e->ev_k[1], &e->ev_o[0], &e->ev_o[1], &e->ev_slot[0], &e->ev_slot[1],
                            &e->ev_slot[2], &e->ev_up[0], &e->ev_up[1], &e->ev_up[2], &e->ev_up[3],
                            &e->ev_used[0], &e->ev_used[1], &e->ev_used[2], &e->ev_used[3], &e->ev_sel[0],
                            &e->ev_sel[1]})
        CK(cudaEventCreateWithFlags(ev, cudaEventDisableTiming));
    Tables t(e->N);
    std::vector<float> w = hann(hop);
    e->tw = dalloc<float2>(t.tw.size());
    e->pk = dalloc<float2>(e->N + 2);
    e->win = dalloc<float>(e->N);
    CK(cudaMemcpy(e->tw, t.tw.data(), sizeof(float2) * t.tw.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(e->pk, t.pk.data(), sizeof(float2) * (e->N + 2), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(e->win, w.data(), sizeof(float) * e->N, cudaMemcpyHostToDevice));
    const size_t ring_elems = (size_t)e->S * 2 * e->D * e->N;
    e->ring = dalloc<float2>(ring_elems);
    e->hist = dalloc<float>((size_t)e->S * e->L);
    e->ola = dalloc<float>((size_t)e->S * e->E * 3 * e->L);
    CK(cudaMemsetAsync(e->ring, 0, ring_elems * sizeof(float2), e->stream));
    CK(cudaMemsetAsync(e->hist, 0, (size_t)e->S * e->L * sizeof(float), e->stream));
    CK(cudaMemsetAsync(e->ola, 0, (size_t)e->S * e->E * 3 * e->L * sizeof(float), e->stream));
    e->sel.assign(e->S, 0);
    e->staged.assign(e->S, 0);
    e->d_sel = dalloc<int>(2 * e->S);
    CK(cudaMemsetAsync(e->d_sel, 0, sizeof(int) * e->S, e->stream));
    for (int b = 0; b < 2; ++b) CK(cudaMallocHost(&e->h_sel[b], sizeof(int) * 2 * e->S));
    apply_default_tuning(e);
    pick_launch_config(e);
    validate_launch(e, e->P, e->NT);
    pick_block_geometry(e);
}

// Device copy of a host/device IR table; returns a device pointer valid on `s`.
const float* stage_ir(tvolap_engine* e, const float* ir, size_t count, cudaStream_t s) {
    if (classify(ir) == Mem::Device) return ir;
    if (e->irstage_cap < count) {
        CK(cudaStreamSynchronize(s));
        if (e->d_irstage) CK(cudaFree(e->d_irstage));
        e->d_irstage = dalloc<float>(count);
        e->irstage_cap = count;
    }
    CK(cudaMemcpyAsync(e->d_irstage, ir, count * sizeof(float), cudaMemcpyHostToDevice, s));
    return e->d_irstage;
}

// Upload a host selection with the sources sorted by it (a stable counting sort over the bank
// entries): the one-hop kernel runs the sources that share an entry in adjacent clusters, so each
// selected filter is read from HBM about once per hop instead of once per source using it.
// Row-pitched copy; one contiguous copy when neither side has gaps between rows (one-hop calls on
// dense [lanes][L] buffers: 4096 rows of 128 B as one 512 KB DMA instead of 4096 descriptors).
cudaError_t copy_rows(void* dst, size_t dpitch, const void* src, size_t spitch, size_t width, size_t rows,
                      cudaMemcpyKind kind, cudaStream_t st) {
    if (dpitch == width && spitch == width) return cudaMemcpyAsync(dst, src, width * rows, kind, st);
    return cudaMemcpy2DAsync(dst, dpitch, src, spitch, width, rows, kind, st);
}

void upload_selection(tvolap_engine* e, const int* sel) {
    const long S = e->S;
    e->sel_dirty = false;
    const int hb = e->sel_next;
    e->sel_next ^= 1;
    CK(cudaEventSynchronize(e->ev_sel[hb]));  // the upload that last read this buffer is done
    int* buf = e->h_sel[hb];
    std::memcpy(buf, sel, sizeof(int) * S);
    e->order_valid = e->entry_order != 0;
    if (e->order_valid) {
        std::vector<int> start(e->n_bank + 1, 0);
        for (long s = 0; s < S; ++s) ++start[sel[s] + 1];
        for (long b = 0; b < e->n_bank; ++b) start[b + 1] += start[b];
        int* order = buf + S;
        for (long s = 0; s < S; ++s) order[start[sel[s]]++] = (int)s;
    }
    CK(cudaMemcpyAsync(e->d_sel, buf, sizeof(int) * (e->order_valid ? 2 : 1) * S, cudaMemcpyHostToDevice,
                       e->stream));
    CK(cudaEventRecord(e->ev_sel[hb], e->stream));
}

void latch(tvolap_engine* e) {  // engine.cpp:54-58
    std::lock_guard<std::mutex> lock(e->mu);
    if (e->pending_ext) {  // a pre-partitioned device set: O(1), read in place from now on
        set_release(e->active_ext);
        e->active_ext = e->pending_ext;
        e->pending_ext = nullptr;
    }
    if (e->pending) {
        set_release(e->active_ext);  // back to the engine's own pool
        e->active_ext = nullptr;
        if (e->staged_on_side) {  // already transformed on the side stream
            CK(cudaStreamWaitEvent(e->stream, e->ev_side, 0));
        } else if (e->staged_in_stream) {  // K4 on the engine stream, chained to the hop launches
            if (e->staged_buf >= 0) CK(cudaStreamWaitEvent(e->stream, e->ev_up[e->staged_buf], 0));
            const int target = (e->active + 1) % kSlots;
            CK(tvb::launch_partition((int)e->L, (int)e->M, e->S, e->staged_ir, e->staged_len, e->staged_len, e->pool,
                                     (long)target * e->S, e->tw, e->pk, e->stream, true));
            ++e->launches;
            if (e->staged_buf >= 0) CK(cudaEventRecord(e->ev_used[e->staged_buf], e->stream));
        } else {  // the first kernel of this call transforms the staged set into the next slot (K4 fused)
            if (e->staged_buf >= 0) CK(cudaStreamWaitEvent(e->stream, e->ev_up[e->staged_buf], 0));
            e->launch_new_ir = e->staged_ir;
            e->launch_new_len = e->staged_len;
            e->launch_buf = e->staged_buf;
        }
        e->active = (e->active + 1) % kSlots;
        e->pending = false;
    }
    if (e->sel_staged) {
        e->sel = e->staged;
        e->sel_dirty = true;
        e->sel_staged = false;
    }
}

// Paths that install further sets into pool slots mid-call (the switching launch, the wide
// pass) need the running filter in a pool slot too: copy an external set into the next slot.
void materialize_ext(tvolap_engine* e) {
    if (!e->active_ext) return;
    const int slot = (e->active + 1) % kSlots;
    const size_t elems = (size_t)e->S * e->M * e->N;
    CK(cudaMemcpyAsync(e->pool + (size_t)slot * elems, e->active_ext->spec, elems * sizeof(float2),
                       cudaMemcpyDeviceToDevice, e->stream));
    e->active = slot;
    set_release(e->active_ext);
    e->active_ext = nullptr;
}

// A replacement staged at the very hop a call starts from supersedes whatever was staged.
void drop_pending(tvolap_engine* e) {
    if (e->pending && e->staged_on_side) CK(cudaStreamWaitEvent(e->stream, e->ev_side, 0));
    e->pending = false;
    set_release(e->pending_ext);
    e->pending_ext = nullptr;
}

void launch_hops(tvolap_engine* e, long hop0, long n, const float* in, long in_stride, float* out, long out_stride,
                 const int* sched, long sched_stride) {
    HopParams p;
    p.L = (int)e->L;
    p.M = (int)e->M;
    p.D = (int)e->D;
    p.S = (int)e->S;
    const bool blocked = n >= e->block_min;
    p.P = blocked ? e->PB : e->P;
    p.hop0 = hop0;
    p.n_hops = (int)n;
    p.in = in;
    p.in_stride = in_stride;
    p.out = out;
    p.out_stride = out_stride;
    p.ring = e->ring;
    p.pool = e->active_ext ? e->active_ext->spec : e->pool;
    if (e->bank && !sched) {  // bank engines without a per-hop schedule: the latched selection
        if (e->sel_dirty) upload_selection(e, e->sel.data());
        sched = e->d_sel;
        sched_stride = 0;
    }
    p.sched = sched;
    p.sched_stride = sched_stride;
    if (!blocked && e->bank && e->entry_order && e->order_valid && sched == e->d_sel && sched_stride == 0)
        p.order = e->d_sel + e->S;
    p.entry_base = (e->bank || e->active_ext) ? 0 : e->active * (int)e->S;
    p.hist = e->hist;
    p.ola = e->ola;
    p.tw = e->tw;
    p.pk = e->pk;
    p.win = e->win;
    p.new_ir = e->launch_new_ir;
    p.new_ir_stride = e->launch_new_len;
    p.new_ir_len = e->launch_new_len;
    p.pool_w = e->pool;
    p.new_entry_base = e->active * (int)e->S;
    p.qm = e->QM;
    p.sw_irs = e->sw_irs_launch;
    p.sw_entry = e->sw_entry_launch;
    p.sw_count = e->sw_count_launch;
    p.sw_period = e->sw_period_launch;
    p.sw_ir_stride = e->sw_len_launch;
    p.sw_ir_len = e->sw_len_launch;
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    if (e->profiling) {
        if (e->prof_used == e->prof_events.size()) {
            cudaEvent_t a, b;
            CK(cudaEventCreate(&a));
            CK(cudaEventCreate(&b));
            e->prof_events.emplace_back(a, b);
        }
        t0 = e->prof_events[e->prof_used].first;
        t1 = e->prof_events[e->prof_used].second;
        ++e->prof_used;
        CK(cudaEventRecord(t0, e->stream));
    }
    if (blocked)
        CK(tvb::launch_block_kernel(p, (int)e->E, e->JH, e->QB, e->NTB, e->stream));
    else if (e->bank && e->hop_ring && (p.ring_var = (int)e->hop_ring, tvb::hop_ring_supported(p, (int)e->E, hop_ring_threads(e)))) {
        CK(tvb::launch_hop_ring_kernel(p, (int)e->E, hop_ring_threads(e), e->stream));
        ++e->ring_launches;
    }
    else
        CK(tvb::launch_hop_kernel(p, (int)e->E, hop_threads(e), e->stream));
    if (t1) CK(cudaEventRecord(t1, e->stream));
    ++e->launches;
    if (!e->bank) CK(cudaEventRecord(e->ev_slot[e->active], e->stream));
    if (e->launch_new_ir) {
        if (e->launch_buf >= 0) CK(cudaEventRecord(e->ev_used[e->launch_buf], e->stream));
        e->launch_new_ir = nullptr;
        e->launch_buf = -1;
    }
}

void ensure_pipeline(tvolap_engine* e, long kc, bool need_sched, bool need_host) {
    if (e->chunk_hops < kc) {
        CK(cudaStreamSynchronize(e->stream));
        CK(cudaStreamSynchronize(e->h2d));
        CK(cudaStreamSynchronize(e->d2h));
        for (int b = 0; b < 2; ++b) {
            if (e->d_in[b]) CK(cudaFree(e->d_in[b]));
            if (e->d_out[b]) CK(cudaFree(e->d_out[b]));
            e->d_in[b] = dalloc<float>((size_t)e->S * kc * e->L);
            e->d_out[b] = dalloc<float>((size_t)e->S * e->E * kc * e->L);
        }
        e->chunk_hops = kc;
    }
    // pinned host staging only for pageable caller buffers (pinned ones are copied directly)
    if (need_host && e->host_chunk < e->chunk_hops) {
        CK(cudaStreamSynchronize(e->h2d));
        CK(cudaStreamSynchronize(e->d2h));
        for (int b = 0; b < 2; ++b) {
            if (e->h_in[b]) CK(cudaFreeHost(e->h_in[b]));
            if (e->h_out[b]) CK(cudaFreeHost(e->h_out[b]));
            CK(cudaMallocHost(&e->h_in[b], sizeof(float) * e->S * e->chunk_hops * e->L));
            CK(cudaMallocHost(&e->h_out[b], sizeof(float) * e->S * e->E * e->chunk_hops * e->L));
        }
        e->host_chunk = e->chunk_hops;
    }
    if (need_sched && e->sch_cap < kc) {
        CK(cudaStreamSynchronize(e->stream));
        for (int b = 0; b < 2; ++b) {
            if (e->d_sch[b]) CK(cudaFree(e->d_sch[b]));
            e->d_sch[b] = dalloc<int>((size_t)e->S * kc);
        }
        e->sch_cap = kc;
    }
}

bool run_wide_bank(tvolap_engine* e, long hop0, const float* in, long in_stride, float* out, long out_stride, long n,
                   const int* sched);
bool run_wide_set(tvolap_engine* e, long hop0, const float* in, long in_stride, float* out, long out_stride, long n);
bool run_bank_pass(tvolap_engine* e, long hop0, const float* in, long in_stride, float* out, long out_stride, long n,
                   const int* dsched);

void process_hops_impl(tvolap_engine* e, const float* in, long in_stride, float* out, long out_stride, long n,
                       const int* sched) {
    CK(cudaSetDevice(e->device));
    latch(e);
    const long L = e->L, S = e->S, E = e->E;
    const Mem min = classify(in), mout = classify(out);
    const Mem msch = sched ? classify(sched) : Mem::Device;
    // a bank schedule that changes rarely (C1): time-parallel passes instead of the hop-blocked launch
    auto hops_launch = [&](long hop0, long kc, const float* ip, long is, float* op, long os, const int* sch_launch,
                           const int* sch_hops) {
        if (sched && e->bank && run_wide_bank(e, hop0, ip, is, op, os, kc, sch_hops)) return;
        if (sched && e->bank && run_bank_pass(e, hop0, ip, is, op, os, kc, sch_launch)) return;
        if (!sched && !e->bank && run_wide_set(e, hop0, ip, is, op, os, kc)) return;
        launch_hops(e, hop0, kc, ip, is, op, os, sch_launch, sched ? S : 0);
    };
    // one hop between pinned host buffers (the reference's process() call from a host that keeps
    // its audio in page-locked memory): the hop kernel reads the hop and writes its outputs through
    // the buffers' device mapping — L floats per source over PCIe while other CTAs multiply —
    // instead of two stream-ordered copies around it
    bool direct = min == Mem::Device && mout == Mem::Device && msch == Mem::Device;
    const float* din = in;
    float* dout = out;
    if (!direct && n == 1 && !sched && e->zero_copy && min != Mem::Pageable && mout != Mem::Pageable) {
        bool ok = true;
        if (min == Mem::Pinned)
            ok = cudaHostGetDevicePointer((void**)&din, const_cast<float*>(in), 0) == cudaSuccess;
        if (ok && mout == Mem::Pinned) ok = cudaHostGetDevicePointer((void**)&dout, out, 0) == cudaSuccess;
        if (ok) {
            direct = true;
        } else {
            cudaGetLastError();
            din = in;
            dout = out;
        }
    }
    if (direct) {
        hops_launch(e->hops, n, din, in_stride, dout, out_stride, sched, sched);
    } else {
        const long per_hop = S * L * (1 + E);
        long kc_want = (1L << e->pipe_log2) / per_hop;
        // bank passes re-read M delay-line slots per pass: chunks of >= 8M hops keep that small
        if (sched && e->bank && e->bank_pass) kc_want = std::max<long>(kc_want, 8 * e->M);
        const long kc_max = std::max<long>(1, std::min<long>(n, kc_want));
        ensure_pipeline(e, kc_max, sched && msch != Mem::Device, min == Mem::Pageable || mout == Mem::Pageable);
        const long Kc = e->chunk_hops;
        // one chunk (one-hop process() calls): nothing to overlap, so the copies go on the engine
        // stream itself — no cross-stream event hand-offs on the latency path
        const bool single = n <= Kc;
        cudaStream_t sh = single ? e->stream : e->h2d, sd = single ? e->stream : e->d2h;
        CK(cudaEventRecord(e->ev_start, e->stream));
        CK(cudaStreamWaitEvent(sh, e->ev_start, 0));
        CK(cudaStreamWaitEvent(sd, e->ev_start, 0));
        struct Pend {
            long h0 = -1, kc = 0;
        } pend[2];
        auto flush_out = [&](int b) {
            if (pend[b].h0 < 0) return;
            CK(cudaEventSynchronize(e->ev_o[b]));
            for (long r = 0; r < S * E; ++r)
                std::memcpy(out + r * out_stride + pend[b].h0 * L, e->h_out[b] + r * Kc * L,
                            sizeof(float) * pend[b].kc * L);
            pend[b].h0 = -1;
        };
        // chunk sizes: full chunks of Kc hops between a ramp up (Kc/32 .. Kc/2, doubling) and the
        // same ramp down, so the first H2D and the last D2H — the only copies no kernel hides — move
        // small chunks; every other copy overlaps the neighbouring chunk's kernels (a 2x step keeps
        // that true while a hop's kernels take >= 2x its copies: C5 ~7x, C3 ~2.3x). Results do not
        // depend on the split (the passes are split-invariant).
        std::vector<long> sizes;
        {
            std::vector<long> ramp;
            for (long k = Kc / 32; k >= 1 && k < Kc; k *= 2)
                if (k >= 16) ramp.push_back(k);
            long rs = 0;
            for (long k : ramp) rs += k;
            long mid = n;
            if (!ramp.empty() && n >= 2 * rs + Kc) {
                sizes = ramp;
                mid = n - 2 * rs;
            }
            for (; mid > 0; mid -= std::min(Kc, mid)) sizes.push_back(std::min(Kc, mid));
            if (sizes.size() > ramp.size() && n >= 2 * rs + Kc) sizes.insert(sizes.end(), ramp.rbegin(), ramp.rend());
        }
        for (long i = 0, h0 = 0; h0 < n; h0 += sizes[(size_t)i++]) {
            const int b = (int)(e->chunk_seq++ & 1);
            const long kc = sizes[(size_t)i];
            const float* in_ptr;
            long in_s;
            const int* sch_ptr = sched ? sched + h0 * S : nullptr;
            bool copied_in = false;
            if (min == Mem::Device) {
                in_ptr = in + h0 * L;
                in_s = in_stride;
            } else {
                CK(cudaStreamWaitEvent(sh, e->ev_k[b], 0));
                if (min == Mem::Pinned) {
                    CK(copy_rows(e->d_in[b], Kc * L * sizeof(float), in + h0 * L, in_stride * sizeof(float),
                                         kc * L * sizeof(float), S, cudaMemcpyHostToDevice, sh));
                } else {
                    CK(cudaEventSynchronize(e->ev_in[b]));
                    for (long r = 0; r < S; ++r)
                        std::memcpy(e->h_in[b] + r * Kc * L, in + r * in_stride + h0 * L, sizeof(float) * kc * L);
                    CK(cudaMemcpyAsync(e->d_in[b], e->h_in[b], sizeof(float) * S * Kc * L, cudaMemcpyHostToDevice,
                                       sh));
                }
                in_ptr = e->d_in[b];
                in_s = Kc * L;
                copied_in = true;
            }
            if (sched && msch != Mem::Device) {
                if (!copied_in) CK(cudaStreamWaitEvent(sh, e->ev_k[b], 0));
                CK(cudaMemcpyAsync(e->d_sch[b], sched + h0 * S, sizeof(int) * S * kc, cudaMemcpyHostToDevice, sh));
                sch_ptr = e->d_sch[b];
                copied_in = true;
            }
            if (copied_in) {
                CK(cudaEventRecord(e->ev_in[b], sh));
                CK(cudaStreamWaitEvent(e->stream, e->ev_in[b], 0));
            }
            float* out_ptr;
            long out_s;
            if (mout == Mem::Device) {
                out_ptr = out + h0 * L;
                out_s = out_stride;
            } else {
                CK(cudaStreamWaitEvent(e->stream, e->ev_o[b], 0));
                out_ptr = e->d_out[b];
                out_s = Kc * L;
            }
            hops_launch(e->hops + h0, kc, in_ptr, in_s, out_ptr, out_s, sch_ptr, sched ? sched + h0 * S : nullptr);
            CK(cudaEventRecord(e->ev_k[b], e->stream));
            if (mout != Mem::Device) {
                CK(cudaStreamWaitEvent(sd, e->ev_k[b], 0));
                if (mout == Mem::Pinned) {
                    CK(copy_rows(out + h0 * L, out_stride * sizeof(float), e->d_out[b], Kc * L * sizeof(float),
                                         kc * L * sizeof(float), S * E, cudaMemcpyDeviceToHost, sd));
                } else {
                    flush_out(b);
                    CK(cudaMemcpyAsync(e->h_out[b], e->d_out[b], sizeof(float) * S * E * Kc * L,
                                       cudaMemcpyDeviceToHost, sd));
                    pend[b].h0 = h0;
                    pend[b].kc = kc;
                }
                CK(cudaEventRecord(e->ev_o[b], sd));
            }
        }
        flush_out(0);
        flush_out(1);
        // later work on the engine stream sees the outputs
        CK(cudaEventRecord(e->ev_start, sd));
        CK(cudaStreamWaitEvent(e->stream, e->ev_start, 0));
    }
    if (sched) {  // the last row becomes the current selection
        std::vector<int> last(S);
        if (msch == Mem::Device) {
            CK(cudaMemcpyAsync(last.data(), sched + (n - 1) * S, sizeof(int) * S, cudaMemcpyDeviceToHost, e->stream));
            CK(cudaStreamSynchronize(e->stream));
        } else {
            std::memcpy(last.data(), sched + (n - 1) * S, sizeof(int) * S);
        }
        e->sel = last;
        e->sel_dirty = true;
    }
    CK(cudaEventRecord(e->ev_main, e->stream));
    e->hops += n;
    e->fwd += (uint64_t)(S * n);
    e->inv += (uint64_t)(S * E * n);
    e->macs += (uint64_t)(S * E * e->M * n);
    const bool pageable = min == Mem::Pageable || mout == Mem::Pageable || msch == Mem::Pageable;
    if (pageable || (!e->host_async && (min != Mem::Device || mout != Mem::Device)))
        CK(cudaStreamSynchronize(e->stream));
}

int check_hops_args(const tvolap_engine* e, const float* in, const float* out, long n) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    if (!in || !out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null input or output buffer");
    if (n < 1) return set_err(TVOLAP_ERR_INVALID_SIZE, "n_hops must be >= 1");
    return TVOLAP_OK;
}

}  // namespace

extern "C" {

const char* tvolap_last_error(void) { return g_err.c_str(); }

const char* tvolap_version(void) { return "tvolap_b200 0.1 (sm_100a)"; }

int tvolap_create(tvolap_engine** out, int device, long hop, long channels, long ir_length, const float* ir,
                  long min_partitions) {
    if (!out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null output handle");
    *out = nullptr;
    // partition.cpp:21-24 checks, in the reference's order
    if (ir_length < 1 || channels < 1 || !ir)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "partition: impulse response is empty");
    if (hop < 2 || !is_pow2(4 * hop))
        return set_err(TVOLAP_ERR_INVALID_SIZE, "partition: 4L must be a power of two, got L = " + std::to_string(hop));
    tvolap_engine* e = nullptr;
    const int rc = guarded([&] {
        require_device(device);
        const long slice = 2 * hop;
        const long M = std::max((ir_length + slice - 1) / slice, std::max<long>(min_partitions, 1));
        e = new tvolap_engine();
        try {
            init_common(e, device, hop, channels, 1, M);
            const size_t slot = (size_t)channels * M * e->N;
            e->pool = dalloc<float2>(kSlots * slot + (size_t)tvb::kWideTail * e->N);  // + rows read by wide prefetches
            CK(cudaMemsetAsync(e->pool, 0, (kSlots * slot + (size_t)tvb::kWideTail * e->N) * sizeof(float2), e->stream));
            const float* src = stage_ir(e, ir, (size_t)channels * ir_length, e->stream);
            CK(tvb::launch_partition((int)hop, (int)M, channels, src, ir_length, ir_length, e->pool, 0, e->tw, e->pk,
                                     e->stream));
            ++e->launches;
            CK(cudaStreamSynchronize(e->stream));
        } catch (...) {
            delete e;
            e = nullptr;
            throw;
        }
    });
    *out = e;
    return rc;
}

int tvolap_create_bank(tvolap_engine** out, int device, long hop, long sources, long ears, long n_bank,
                       long ir_length, const float* bank_ir, long min_partitions) {
    if (!out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null output handle");
    *out = nullptr;
    if (ir_length < 1 || sources < 1 || n_bank < 1 || !bank_ir)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "partition: impulse response is empty");
    if (ears < 1 || ears > 2) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "ears must be 1 or 2");
    if (hop < 2 || !is_pow2(4 * hop))
        return set_err(TVOLAP_ERR_INVALID_SIZE, "partition: 4L must be a power of two, got L = " + std::to_string(hop));
    tvolap_engine* e = nullptr;
    const int rc = guarded([&] {
        require_device(device);
        const long slice = 2 * hop;
        const long M = std::max((ir_length + slice - 1) / slice, std::max<long>(min_partitions, 1));
        // the bank kernels address the spectra with 32-bit float4 offsets (<= 64 GB of spectra)
        if ((double)n_bank * ears * M * hop >= 4294967296.0)
            throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "bank too large (over 2^32 float4 of spectra)"};
        e = new tvolap_engine();
        try {
            init_common(e, device, hop, sources, ears, M);
            e->bank = true;
            e->n_bank = n_bank;
            pick_block_geometry(e);
            const long rows = n_bank * ears;
            e->pool = dalloc<float2>((size_t)rows * M * e->N + (size_t)tvb::kWideTail * e->N);  // + rows read by wide prefetches
            const float* src = stage_ir(e, bank_ir, (size_t)rows * ir_length, e->stream);
            CK(tvb::launch_partition((int)hop, (int)M, rows, src, ir_length, ir_length, e->pool, 0, e->tw, e->pk,
                                     e->stream));
            ++e->launches;
            CK(cudaStreamSynchronize(e->stream));
        } catch (...) {
            delete e;
            e = nullptr;
            throw;
        }
    });
    *out = e;
    return rc;
}

int tvolap_destroy(tvolap_engine* e) {
    delete e;
    return TVOLAP_OK;
}

// Host schedules are range-checked before anything runs (an index past the bank would be read out
// of bounds on the device). A branch-free unsigned compare the compiler vectorises, split over host
// threads for large schedules (C5: 61 M entries per 10-s call took ~50 ms as an early-exit loop).
bool schedule_in_range(const int32_t* s, long n, long n_bank) {
    auto part = [&](long a, long b) {
        unsigned bad = 0;
        for (long i = a; i < b; ++i) bad |= (unsigned)s[i] >= (unsigned)n_bank;
        return bad == 0;
    };
    const long T = n < (1L << 22) ? 1 : std::min<long>(16, std::max(1u, std::thread::hardware_concurrency()));
    if (T == 1) return part(0, n);
    std::vector<char> ok((size_t)T, 1);
    std::vector<std::thread> th;
    for (long t = 0; t < T; ++t)
        th.emplace_back([&, t] { ok[(size_t)t] = part(n * t / T, n * (t + 1) / T) ? 1 : 0; });
    for (auto& x : th) x.join();
    for (char c : ok)
        if (!c) return false;
    return true;
}

int tvolap_process(tvolap_engine* e, const float* in, long in_lane_stride, long rows, long cols, float* out,
                   long out_lane_stride) {
    if (int rc = check_hops_args(e, in, out, 1)) return rc;
    if (rows != e->L || cols != e->S) {
        // the reference latches a staged filter before its shape checks (engine.cpp:61-67)
        if (int rc = guarded([&] {
                CK(cudaSetDevice(e->device));
                latch(e);
            }))
            return rc;
        if (rows != e->L)
            return set_err(TVOLAP_ERR_INVALID_SIZE, "process() expects exactly one hop of input per call");
        return set_err(TVOLAP_ERR_INVALID_INPUT, "input channel count does not match the filter");
    }
    return guarded([&] { process_hops_impl(e, in, in_lane_stride, out, out_lane_stride, 1, nullptr); });
}

int tvolap_process_hops(tvolap_engine* e, const float* in, long in_lane_stride, float* out, long out_lane_stride,
                        long n_hops, const int32_t* schedule) {
    if (int rc = check_hops_args(e, in, out, n_hops)) return rc;
    if (schedule && !e->bank)
        return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "a bank schedule needs a bank engine");
    if (in_lane_stride < n_hops * e->L || out_lane_stride < n_hops * e->L)
        return set_err(TVOLAP_ERR_INVALID_SIZE, "lane stride shorter than n_hops * L");
    if (schedule && classify(schedule) != Mem::Device && !schedule_in_range(schedule, n_hops * e->S, e->n_bank))
        return set_err(TVOLAP_ERR_INVALID_INPUT, "bank index out of range in schedule");
    return guarded([&] { process_hops_impl(e, in, in_lane_stride, out, out_lane_stride, n_hops, schedule); });
}

// ---- time-parallel pass (tvolap_wide.cu) for device-resident switching calls
extern "C++" {
namespace {

int sm_count_of(int device) {
    int sms = 148;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
    return sms;
}

// The period tiles of wide_period_kernel apply: every period one tile of <= 8 hops with its set
// transformed in shared-memory partition groups (C4).
bool period_tiles(const tvolap_engine* e, long period, long ir_length) {
    return e->wide_period != 0 && e->wide_fuse != 0 && e->wide_warp_fft != 0 && period >= 3 && period <= 8 &&
           tvb::period_kernel_supported((int)e->L, (int)e->M, 4, ir_length);
}

bool wide_eligible(const tvolap_engine* e, long n_hops, long period, long ir_length) {
    if (e->wide_mode == 0 || e->bank || e->E != 1 || !tvb::wide_supported((int)e->L)) return false;
    if (period < 3 || n_hops < period || n_hops < 16) return false;
    // auto: where the hop-blocked kernel leaves most of the GPU idle (lanes x cluster CTAs below
    // two per SM, e.g. C1/C2; there the hop axis is the parallelism), or where the period tiles
    // keep every set's spectra on chip (C4)
    if (e->wide_mode == 1 && e->S * e->PB > 2 * e->sms && !period_tiles(e, period, ir_length)) return false;
    return true;
}

void prof_pair(tvolap_engine* e, cudaEvent_t* t0, cudaEvent_t* t1) {
    *t0 = *t1 = nullptr;
    if (!e->profiling) return;
    if (e->prof_used == e->prof_events.size()) {
        cudaEvent_t a, b;
        CK(cudaEventCreate(&a));
        CK(cudaEventCreate(&b));
        e->prof_events.emplace_back(a, b);
    }
    *t0 = e->prof_events[e->prof_used].first;
    *t1 = e->prof_events[e->prof_used].second;
    ++e->prof_used;
}

template <class T>
void ensure_dev(T*& p, size_t& cap, size_t count) {
    if (cap >= count) return;
    if (p) CK(cudaFree((void*)p));
    p = dalloc<std::remove_const_t<T>>(count);
    cap = count;
}

// One time-parallel pass over nh hops starting at the engine's current hop: tiles t0 (starts,
// nh appended), filter sets fs per tile (base of [S][M][2L]) or, with per_lane, per (tile, lane)
// (base of [M][2L]); tirs (optional): per tile the IR set the tile transforms itself (fused K4).
void wide_pass(tvolap_engine* e, long hop0, const float* in, long in_stride, float* out, long out_stride, long nh,
               const std::vector<int>& t0, const std::vector<const float2*>& fs, bool per_lane,
               const std::vector<const float*>* tirs, long ir_length, int JH, int nslots, int warp_fft,
               int period_smem = 0) {
    const long S = e->S, M = e->M, N = e->N, L = e->L;
    const long ntiles = (long)t0.size() - 1;
    ensure_dev(e->d_wide_fset, e->wide_fset_cap, fs.size());
    ensure_dev(e->d_wide_tile0, e->wide_tile_cap, (size_t)ntiles + 1);
    CK(cudaMemcpyAsync(e->d_wide_fset, fs.data(), sizeof(const float2*) * fs.size(), cudaMemcpyHostToDevice,
                       e->stream));
    CK(cudaMemcpyAsync(e->d_wide_tile0, t0.data(), sizeof(int) * (ntiles + 1), cudaMemcpyHostToDevice, e->stream));
    if (tirs) {
        ensure_dev(e->d_wide_tile_ir, e->wide_tile_ir_cap, (size_t)ntiles);
        CK(cudaMemcpyAsync(e->d_wide_tile_ir, tirs->data(), sizeof(const float*) * ntiles, cudaMemcpyHostToDevice,
                           e->stream));
    }
    // carry and head terms per tile, extended spectra
    ensure_dev(e->wide_state, e->wide_state_cap, (size_t)S * ntiles * 3 * L);
    ensure_dev(e->wide_head, e->wide_head_cap, (size_t)S * ntiles * 6 * L);
    const long T = (nh + 1) / 2 + M + tvb::kWideFront + JH + 4;
    ensure_dev(e->wide_xe, e->wide_xe_cap, (size_t)S * 2 * T * N);
    tvb::WideParams p{};
    p.L = (int)L;
    p.M = (int)M;
    p.D = (int)e->D;
    p.S = (int)S;
    // partition groups: the hop-blocked kernel's (bit-identical sums) with its Stockham transforms;
    // one chain with the warp transforms (equal to fp32 rounding anyway; TVOLAP_WIDE_Q overrides)
    p.Q = e->wide_q > 0 ? (int)e->wide_q : (warp_fft ? 1 : e->QM);
    p.hop0 = hop0;
    p.n = (int)nh;
    p.in = in;
    p.in_stride = in_stride;
    p.out = out;
    p.out_stride = out_stride;
    p.ring = e->ring;
    p.xe = e->wide_xe;
    p.T = T;
    p.tbase = (hop0 >> 1) - M - tvb::kWideFront;
    p.hist = e->hist;
    p.ola = e->ola;
    p.tw = e->tw;
    p.pk = e->pk;
    p.win = e->win;
    p.fset = e->d_wide_fset;
    p.fset_per_lane = per_lane ? 1 : 0;
    p.tile0 = e->d_wide_tile0;
    p.ntiles = (int)ntiles;
    p.tstate = e->wide_state;
    p.thead = e->wide_head;
    p.tile_ir = tirs ? e->d_wide_tile_ir : nullptr;
    p.ir_len = ir_length;
    p.scratch = e->wide_scratch;
    p.slot_lock = e->wide_lock;
    p.nslots = nslots;
    p.warp_fft = warp_fft;
    p.k1_small = (int)e->k1_small;
    p.stage_ir = (int)e->wide_stage;
    p.period_smem = period_smem;
    cudaEvent_t ev0, ev1;
    prof_pair(e, &ev0, &ev1);
    CK(tvb::launch_wide(p, JH, e->stream, ev0, ev1, 3));
    e->launches += 4;
    ++e->wide_passes;
}

// The call as time-parallel passes (chunks of periods whose new sets fit the pool budget): K4
// of the chunk's sets, K1 of all its hops, then (lane, tile) CTAs for K3+K5 and the OLA fix-up.
// Same results, bit for bit, as the switching / hop-blocked launches.
void run_wide(tvolap_engine* e, const float* in, long in_stride, float* out, long out_stride, long n_hops,
              long period, const float* const* irs, long ir_length) {
    const long S = e->S, M = e->M, N = e->N, L = e->L;
    const long nsw = (n_hops + period - 1) / period;
    const long last = n_hops - (nsw - 1) * period;
    const long nsw_w = last >= 3 ? nsw : nsw - 1;  // a 1-2 hop final period runs on the blocked path
    const long n_w = last >= 3 ? n_hops : (nsw - 1) * period;
    if (irs[0]) {  // a staged set is superseded at this very hop (last wins)
        std::lock_guard<std::mutex> lock(e->mu);
        drop_pending(e);
    }
    latch(e);
    materialize_ext(e);
    if (e->launch_new_ir) {  // a latched set the first hop launch would have transformed (fused-K4 mode)
        CK(tvb::launch_partition((int)L, (int)M, S, e->launch_new_ir, e->launch_new_len, e->launch_new_len, e->pool,
                                 (long)e->active * S, e->tw, e->pk, e->stream));
        ++e->launches;
        if (e->launch_buf >= 0) CK(cudaEventRecord(e->ev_used[e->launch_buf], e->stream));
        e->launch_new_ir = nullptr;
        e->launch_buf = -1;
    }
    // 16-hop tiles, or 8-hop tiles when no period needs more (8-hop periods would leave half of a
    // 16-hop tile's MAC outputs unused) or the 16-hop tile's shared memory does not fit
    int JH = period <= 8 ? 4 : 8;
    if (tvb::wide_mac_smem_bytes((int)L, JH, (int)M, e->QM) > 227 * 1024) JH = 4;
    const long Jmax = 2 * JH;
    const size_t set_elems = (size_t)S * M * N;
    const long budget_mb = e->wide_pool_mb;
    const long cap_sets = std::max<long>(1, (long)((budget_mb << 20) / (long)(set_elems * sizeof(float2))));
    const float2* cur_set = e->pool + (size_t)e->active * set_elems;
    // Fused K4: when every period is one tile, each tile transforms its own set into an
    // L2-resident scratch slot (no set spectra through HBM); TVOLAP_WIDE_FUSE=0 disables.
    const bool fuse = e->wide_fuse != 0 && period <= Jmax && period >= 3;
    // period tiles: the set of each tile transformed group by group into shared memory (the IR
    // slices arrive by bulk copies: 16-byte aligned sets)
    bool ptiles = fuse && JH == 4 && period_tiles(e, period, ir_length);
    for (long k = 0; ptiles && k < nsw; ++k) ptiles = !irs[k] || (reinterpret_cast<uintptr_t>(irs[k]) & 15) == 0;
    int nslots = 0;
    if (fuse && !ptiles) {
        const int q_launch = e->wide_q > 0 ? (int)e->wide_q : (e->wide_warp_fft ? 1 : e->QM);  // as wide_pass sets it
        nslots = tvb::wide_mac_ctas_per_sm((int)L, JH, (int)M, q_launch) * sm_count_of(e->device);
        if (nslots <= 0) throw ApiError{TVOLAP_ERR_CUDA, "wide pass: no resident CTA for the MAC kernel"};
        ensure_dev(e->wide_scratch, e->wide_scratch_cap, (size_t)nslots * (M + tvb::kWideTail) * N);
        if (e->wide_lock_cap < (size_t)nslots) {
            ensure_dev(e->wide_lock, e->wide_lock_cap, (size_t)nslots);
            CK(cudaMemsetAsync(e->wide_lock, 0, sizeof(unsigned) * nslots, e->stream));
        }
    }
    const float* cur_ir = nullptr;  // fused: the IR set in effect (null: the engine's active set)
    const float* last_ir = nullptr;
    // periods per pass: the extended spectra (and per-tile carries) of a pass stay within
    // TVOLAP_WIDE_XE_MB (default 4 GB), the sets of an unfused pass within TVOLAP_WIDE_POOL_MB
    const long xe_mb = e->wide_xe_mb;
    const long per_period = (long)(S * N * sizeof(float2) * period + S * 9 * L * sizeof(float));
    const long cap_periods = std::max<long>(1, (xe_mb << 20) / std::max<long>(1, per_period) - (M + 32) / period);
    for (long k0 = 0; k0 < nsw_w;) {
        long k1 = k0, nsets = 0;
        while (k1 < nsw_w && k1 - k0 < cap_periods && (fuse || !irs[k1] || nsets < cap_sets))
            nsets += (irs[k1++] && !fuse) ? 1 : 0;
        const long h0 = k0 * period, nh = std::min(k1 * period, n_w) - h0;
        // K4 for the chunk's sets
        std::vector<const float*> tab;
        for (long k = k0; k < k1; ++k)
            if (irs[k]) tab.push_back(irs[k]);
        if (nsets) {
            ensure_dev(e->wide_pool, e->wide_pool_cap, (size_t)nsets * set_elems + (size_t)tvb::kWideTail * N);
            ensure_dev(e->d_wide_irs, e->wide_sw_cap, (size_t)nsets);
            CK(cudaMemcpyAsync(e->d_wide_irs, tab.data(), sizeof(const float*) * nsets, cudaMemcpyHostToDevice,
                               e->stream));
            CK(tvb::launch_partition_multi((int)L, (int)M, (int)S, nsets * S, e->d_wide_irs, ir_length, e->wide_pool,
                                           e->tw, e->pk, e->stream));
            ++e->launches;
        }
        // tiles: each period split into balanced tiles of <= 2 JH hops (>= 3 each: OLA fix-up)
        std::vector<int> t0;
        std::vector<const float2*> fs;
        std::vector<const float*> tirs;
        long idx = 0;
        for (long k = k0; k < k1; ++k) {
            if (irs[k] && !fuse) cur_set = e->wide_pool + (size_t)(idx++) * set_elems;
            if (irs[k] && fuse) cur_ir = last_ir = irs[k];
            tirs.push_back(cur_ir);
            const long plen = std::min(period, n_w - k * period);
            const long tp = (plen + Jmax - 1) / Jmax, base = plen / tp, rem = plen % tp;
            long st = k * period - h0;
            for (long w = 0; w < tp; ++w) {
                t0.push_back((int)st);
                fs.push_back(cur_set);
                st += base + (w < rem ? 1 : 0);
            }
        }
        t0.push_back((int)nh);
        if (fuse && tirs.size() != fs.size())
            throw ApiError{TVOLAP_ERR_CUDA, "wide pass: fused K4 needs one tile per period"};
        wide_pass(e, e->hops, in + h0 * L, in_stride, out + h0 * L, out_stride, nh, t0, fs, false,
                  fuse ? &tirs : nullptr, ir_length, JH, nslots, e->wide_warp_fft, ptiles ? 1 : 0);
        e->hops += nh;
        if (fuse && last_ir) {  // the pass's last set becomes the engine's active set (K4 into a pool slot)
            const int slot = (e->active + 1) % kSlots;
            CK(tvb::launch_partition((int)L, (int)M, S, last_ir, ir_length, ir_length, e->pool, (long)slot * S, e->tw,
                                     e->pk, e->stream));
            ++e->launches;
            e->active = slot;
            cur_set = e->pool + (size_t)slot * set_elems;
        }
        if (nsets) {  // the chunk's last set becomes the engine's active set (a pool slot)
            const int slot = (e->active + 1) % kSlots;
            float2* dst = e->pool + (size_t)slot * set_elems;
            CK(cudaMemcpyAsync(dst, cur_set, set_elems * sizeof(float2), cudaMemcpyDeviceToDevice, e->stream));
            e->active = slot;
            cur_set = dst;
        }
        k0 = k1;
    }
    for (int i = 0; i < kSlots; ++i) CK(cudaEventRecord(e->ev_slot[i], e->stream));
    CK(cudaEventRecord(e->ev_main, e->stream));
    e->fwd += (uint64_t)(S * n_w);
    e->inv += (uint64_t)(S * n_w);
    e->macs += (uint64_t)(S * M * n_w);
    if (n_w < n_hops) {  // final 1-2 hop period: the blocked path with its set
        if (irs[nsw - 1]) {
            const int rc = tvolap_exchange_filter(e, irs[nsw - 1], ir_length, S);
            if (rc) throw ApiError{rc, g_err};
        }
        process_hops_impl(e, in + n_w * L, in_stride, out + n_w * L, out_stride, n_hops - n_w, nullptr);
    }
}


// Bank engines with a per-hop schedule that changes rarely (C1: two IRs alternating every 64
// hops) on device buffers: time-parallel passes with tiles that never straddle a change of any
// lane's entry, each tile reading its lanes' bank entries in place. The hop kernels' Stockham
// transforms keep it bit-identical to the hop-blocked launch (process_hops == process()).
// Returns false (nothing done) when the engine or schedule does not qualify. `sched` may be host or
// device memory; hop0 is the global index of the call's first hop.
bool run_wide_bank(tvolap_engine* e, long hop0, const float* in, long in_stride, float* out, long out_stride, long n,
                   const int* sched) {
    const long S = e->S, M = e->M, N = e->N, L = e->L;
    if (e->wide_mode == 0 || e->E != 1 || !tvb::wide_supported((int)L) || n < 16) return false;
    if (e->wide_mode == 1 && e->S * e->PB > 2 * e->sms) return false;
    std::vector<int> h((size_t)n * S);
    if (classify(sched) == Mem::Device) {
        CK(cudaMemcpyAsync(h.data(), sched, sizeof(int) * h.size(), cudaMemcpyDeviceToHost, e->stream));
        CK(cudaStreamSynchronize(e->stream));
    } else {
        std::memcpy(h.data(), sched, sizeof(int) * h.size());
    }
    // segments: maximal hop ranges over which no lane changes its entry; all >= 3 hops
    std::vector<long> seg{0};
    for (long k = 1; k < n; ++k)
        if (std::memcmp(&h[(size_t)k * S], &h[(size_t)(k - 1) * S], sizeof(int) * S) != 0) seg.push_back(k);
    seg.push_back(n);
    long longest = 0;
    for (size_t i = 0; i + 1 < seg.size(); ++i) {
        if (seg[i + 1] - seg[i] < 3) return false;
        longest = std::max(longest, seg[i + 1] - seg[i]);
    }
    for (int v : h)
        if (v < 0 || v >= e->n_bank) return false;  // validated by the caller; never read outside the bank
    int JH = longest <= 8 ? 4 : 8;
    if (tvb::wide_mac_smem_bytes((int)L, JH, (int)M, e->QM) > 227 * 1024) JH = 4;
    const long Jmax = 2 * JH;
    const long xe_mb = e->wide_xe_mb;
    const long max_hops = std::max<long>(Jmax, (xe_mb << 20) / (long)(S * N * sizeof(float2)) - 2 * (M + 32));
    const size_t entry_elems = (size_t)e->E * M * N;
    for (size_t i0 = 0; i0 + 1 < seg.size();) {  // passes of whole segments
        size_t i1 = i0 + 1;
        while (i1 + 1 < seg.size() && seg[i1 + 1] - seg[i0] <= max_hops) ++i1;
        const long h0 = seg[i0], nh = seg[i1] - h0;
        std::vector<int> t0;
        std::vector<const float2*> fs;
        for (size_t i = i0; i < i1; ++i) {
            const long plen = seg[i + 1] - seg[i];
            const long tp = (plen + Jmax - 1) / Jmax, base = plen / tp, rem = plen % tp;
            long st = seg[i] - h0;
            for (long w = 0; w < tp; ++w) {
                t0.push_back((int)st);
                for (long s = 0; s < S; ++s) fs.push_back(e->pool + (size_t)h[(size_t)seg[i] * S + s] * entry_elems);
                st += base + (w < rem ? 1 : 0);
            }
        }
        t0.push_back((int)nh);
        wide_pass(e, hop0 + h0, in + h0 * L, in_stride, out + h0 * L, out_stride, nh, t0, fs, true, nullptr, 0, JH, 0,
                  0);
        i0 = i1;
    }
    return true;  // (the caller accounts hops, counts and the latched selection)
}

// Bank engines with a per-hop schedule that changes every hop (C3, C5) on device-resident hops
// (the whole call, or one chunk of the pinned-host pipeline): bank passes (tvolap_wide.cu) — K1
// of every hop into Xe, the MAC over (tile, source, partition group) CTAs with the group as the
// slowest grid axis (the bank slice each group reads stays L2-resident), K5 + overlap-add per
// (tile, output lane) and the carry fix-up. `dsched` is device memory (rows of the call's hops).
// Not bit-identical to the hop-blocked kernel (different partition grouping and transforms);
// both match the reference within the north-star tolerance. False when not eligible.
bool run_bank_pass(tvolap_engine* e, long hop0, const float* in, long in_stride, float* out, long out_stride, long n,
                   const int* dsched) {
    const long S = e->S, M = e->M, N = e->N, L = e->L, E = e->E;
    if (!e->bank_pass || !dsched || classify(dsched) != Mem::Device) return false;
    // tiles of 64 hops (one CTA of 512 threads per SM) where the register budget allows: fewer Xe
    // window rows per output than 32-hop tiles (C5 1.94e9 -> 1.97e9; -> 2.02e9 with every CTA
    // walking all tiles of its (source, group), so the window stays in L1: profiles/r02_ab_bank_tpc.txt)
    // two ears: 32-hop tiles where the K5 tile fits (C3 7.13e9 -> 7.18e9)
    int JH = (N <= 128 && E == 1) ? 32 : (E == 2 && N <= 256) ? 16 : 8;
    if (e->bank_pass_jh > 0 && tvb::bank_pass_supported((int)L, (int)E, (int)e->bank_pass_jh)) JH = (int)e->bank_pass_jh;
    const long J = 2 * JH;
    // (any call of >= 3 hops: the same per-output sums whatever the call / chunk boundaries)
    if (!tvb::bank_pass_supported((int)L, (int)E, JH) || n < 3) return false;
    // partition groups: the fewest whose bank slice stays well inside L2 (<= 40 MB); fewer groups
    // = fewer partial sums through HBM (C5: Q = 7, 38 MB slices, 1.89e9 vs 1.86e9 with Q = 8 and
    // 1.77e9 with Q = 4, profiles/r02_ab_bank_q.txt)
    const double bank_bytes = (double)e->n_bank * E * M * N * sizeof(float2);
    int Q = (int)std::min<long>(std::min<long>(64, M), std::max<long>(1, (long)std::ceil(bank_bytes / 40e6)));
    if (e->bank_pass_q > 0) Q = (int)std::min<long>(e->bank_pass_q, M);
    // hops per pass: extended spectra + partials within the budget
    const long per_hop = (long)(S * N * sizeof(float2) + (size_t)Q * S * E * N * sizeof(float2));
    long max_hops = std::max<long>(4 * J, (e->bank_pass_mb << 20) / per_hop);
    max_hops -= max_hops % J;  // whole tiles per pass
    if (e->bank_pass_hops > 0) max_hops = std::max<long>(2 * J, e->bank_pass_hops);
    for (long h0 = 0; h0 < n;) {
        long nh = std::min(max_hops, n - h0);
        if (n - h0 - nh > 0 && n - h0 - nh < 3) nh -= 3;  // no 1-2 hop pass at the end
        // full J-hop tiles and one shorter last tile (whose idle MAC warps exit at once); a 1-2 hop
        // remainder borrows from the tile before it, so every tile has 3 .. J hops
        std::vector<int> t0;
        for (long st = 0; st < nh;) {
            t0.push_back((int)st);
            long len = std::min<long>(J, nh - st);
            if (nh - st - len > 0 && nh - st - len < 3) len -= 3 - (nh - st - len);
            st += len;
        }
        t0.push_back((int)nh);
        const long ntiles = (long)t0.size() - 1;
        ensure_dev(e->d_wide_tile0, e->wide_tile_cap, (size_t)ntiles + 1);
        CK(cudaMemcpyAsync(e->d_wide_tile0, t0.data(), sizeof(int) * (ntiles + 1), cudaMemcpyHostToDevice, e->stream));
        ensure_dev(e->wide_state, e->wide_state_cap, (size_t)S * E * ntiles * 3 * L);
        ensure_dev(e->wide_head, e->wide_head_cap, (size_t)S * E * ntiles * 6 * L);
        const long T = (nh + 1) / 2 + M + tvb::kWideFront + JH + 4;
        ensure_dev(e->wide_xe, e->wide_xe_cap, (size_t)S * 2 * T * N);
        ensure_dev(e->bank_yq, e->bank_yq_cap, (size_t)Q * S * E * nh * N);
        tvb::WideParams p{};
        p.L = (int)L;
        p.M = (int)M;
        p.D = (int)e->D;
        p.S = (int)S;
        p.Q = Q;
        p.E = (int)E;
        p.hop0 = hop0 + h0;
        p.n = (int)nh;
        p.in = in + h0 * L;
        p.in_stride = in_stride;
        p.out = out + h0 * L;
        p.out_stride = out_stride;
        p.ring = e->ring;
        p.xe = e->wide_xe;
        p.T = T;
        p.tbase = (p.hop0 >> 1) - M - tvb::kWideFront;
        p.hist = e->hist;
        p.ola = e->ola;
        p.tw = e->tw;
        p.pk = e->pk;
        p.win = e->win;
        p.tile0 = e->d_wide_tile0;
        p.ntiles = (int)ntiles;
        p.tstate = e->wide_state;
        p.thead = e->wide_head;
        p.warp_fft = 1;
        p.k1_small = (int)e->k1_small;
        p.tpc = e->bank_pass_tpc > 0 ? (int)std::min<long>(e->bank_pass_tpc, ntiles) : (int)ntiles;
        p.pool = e->pool;
        p.sched = dsched + h0 * S;
        p.yq = e->bank_yq;
        cudaEvent_t ev0, ev1;
        prof_pair(e, &ev0, &ev1);
        CK(tvb::launch_bank_pass(p, JH, e->stream, ev0, ev1));
        e->launches += 5;
        ++e->wide_passes;
        h0 += nh;
    }
    return true;  // (the caller accounts hops, counts and the latched selection)
}

// Filter-set engines: a process_hops call (one filter for all its hops) on device buffers or a
// pinned-pipeline chunk as one time-parallel pass over the active set, with the hop kernels'
// Stockham transforms (bit-identical to the hop-blocked launch). False when not eligible.
bool run_wide_set(tvolap_engine* e, long hop0, const float* in, long in_stride, float* out, long out_stride, long n) {
    const long S = e->S, M = e->M, N = e->N, L = e->L;
    if (e->wide_mode == 0 || e->E != 1 || !tvb::wide_supported((int)L) || n < 32) return false;
    if (e->wide_mode == 1 && e->S * e->PB > 2 * e->sms) return false;
    if (e->launch_new_ir) return false;  // a staged set the first hop launch transforms (K4 fused mode)
    int JH = 8;
    if (tvb::wide_mac_smem_bytes((int)L, JH, (int)M, e->QM) > 227 * 1024) JH = 4;
    const long Jmax = 2 * JH;
    const long xe_mb = e->wide_xe_mb;
    const long max_hops = std::max<long>(Jmax, (xe_mb << 20) / (long)(S * N * sizeof(float2)) - 2 * (M + 32));
    const float2* set = e->active_ext ? e->active_ext->spec : e->pool + (size_t)e->active * S * M * N;
    for (long h0 = 0; h0 < n;) {
        long nh = std::min(max_hops, n - h0);
        if (n - h0 - nh > 0 && n - h0 - nh < 3) nh -= 3;  // no 1-2 hop pass at the end
        const long tp = (nh + Jmax - 1) / Jmax, base = nh / tp, rem = nh % tp;
        std::vector<int> t0;
        std::vector<const float2*> fs;
        long st = 0;
        for (long w = 0; w < tp; ++w) {
            t0.push_back((int)st);
            fs.push_back(set);
            st += base + (w < rem ? 1 : 0);
        }
        t0.push_back((int)nh);
        wide_pass(e, hop0 + h0, in + h0 * L, in_stride, out + h0 * L, out_stride, nh, t0, fs, false, nullptr, 0, JH, 0,
                  0);
        h0 += nh;
    }
    CK(cudaEventRecord(e->ev_slot[e->active], e->stream));  // the last reader of the active slot
    return true;
}
}  // namespace
}  // extern "C++"

int tvolap_process_switching(tvolap_engine* e, const float* in, long in_lane_stride, float* out, long out_lane_stride,
                             long n_hops, long period, const float* const* irs, long ir_length) {
    if (int rc = check_hops_args(e, in, out, n_hops)) return rc;
    if (e->bank) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "process_switching needs a filter-set engine");
    if (period < 1) return set_err(TVOLAP_ERR_INVALID_SIZE, "switch period must be >= 1 hop");
    if (!irs) return set_err(TVOLAP_ERR_INVALID_INPUT, "null IR list");
    if (in_lane_stride < n_hops * e->L || out_lane_stride < n_hops * e->L)
        return set_err(TVOLAP_ERR_INVALID_SIZE, "lane stride shorter than n_hops * L");
    const long nsw = (n_hops + period - 1) / period;
    bool any = false;
    for (long k = 0; k < nsw; ++k) any |= irs[k] != nullptr;
    if (any && ir_length < 1) return set_err(TVOLAP_ERR_INVALID_INPUT, "partition: impulse response is empty");
    if (any && (ir_length + 2 * e->L - 1) / (2 * e->L) > e->M)
        return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter partition count differs");
    return guarded([&] {
        CK(cudaSetDevice(e->device));
        {  // device-resident call with enough hops: the time-parallel pass
            bool wide = classify(in) == Mem::Device && classify(out) == Mem::Device && wide_eligible(e, n_hops, period, ir_length);
            for (long k = 0; wide && k < nsw; ++k) wide = !irs[k] || classify(irs[k]) == Mem::Device;
            if (wide) {
                run_wide(e, in, in_lane_stride, out, out_lane_stride, n_hops, period, irs, ir_length);
                return;
            }
        }
        // In-kernel K4 pays off when a CTA's share of one switch's partitions fits the barrier gaps
        // of a period (2 gaps per block, one partition per warp each): C2 16 partitions per CTA in
        // one 16-hop block -> 2.37 vs 2.83 us/hop; C4 (2048-point, 32 per CTA per 8-hop period)
        // is faster as the loop with the in-stream K4 launch.
        const long J = 2L * e->JH, blocks = (period + J - 1) / J;
        const long units = (e->M + e->PB - 1) / e->PB, warps = e->NTB / 32;
        const Mem min = classify(in), mout = classify(out);
        bool dev = min == Mem::Device && mout == Mem::Device && n_hops >= e->block_min;
        bool pinned = min == Mem::Pinned && mout == Mem::Pinned;
        // the switching kernel (in-kernel K4); in a pinned pipeline every chunk launch must take
        // the hop-blocked kernel: full periods, and a last one of at least block_min hops
        const long gap_units = 2 * warps * blocks * e->k4_gap_mult;
        const bool n_ok = e->N == 256 || e->N == 512 || (e->N == 1024 && e->sw_1024);
        const bool kernel_ok = n_ok && e->E == 1 && units <= gap_units &&
                               (!pinned || (period >= e->block_min && n_hops - (nsw - 1) * period >= e->block_min));
        dev = dev && kernel_ok;
        for (long k = 0; k < nsw; ++k) {
            const Mem mk = irs[k] ? classify(irs[k]) : (dev ? Mem::Device : Mem::Pinned);
            dev = dev && mk == Mem::Device;
            pinned = pinned && mk == Mem::Pinned;
        }
        if (!dev && !pinned) {  // the loop it stands for (device buffers without the kernel, pageable)
            for (long k = 0; k < nsw; ++k) {
                const long h0 = k * period, kc = std::min(period, n_hops - h0);
                if (irs[k]) {
                    const int rc = tvolap_exchange_filter(e, irs[k], ir_length, e->S);
                    if (rc) throw ApiError{rc, g_err};
                }
                process_hops_impl(e, in + h0 * e->L, in_lane_stride, out + h0 * e->L, out_lane_stride, kc, nullptr);
            }
            return;
        }
        if (kernel_ok && irs[0]) {  // a staged set is superseded at this very hop (last wins)
            std::lock_guard<std::mutex> lock(e->mu);
            drop_pending(e);
        }
        if (kernel_ok) {
            latch(e);
            materialize_ext(e);
        }
        const long S = e->S, L = e->L;
        // Host pipeline (pinned buffers): chunks of Kp periods staged through two device buffers;
        // H2D of chunk c+1 and D2H of chunk c-1 overlap the launch of chunk c, every copy large.
        long Kp = nsw;
        if (pinned) {
            const long per = S * period * L * 4 * 2 + (ir_length > 0 ? S * ir_length * 4 : 0);
            Kp = std::max<long>(1, std::min<long>(nsw, (e->pipe_mb << 20) / per));
        }
        std::vector<const float*> ptrs(nsw);
        std::vector<int> entries(nsw, -1);
        int slot = e->active;
        for (long k = 0; k < nsw; ++k) {
            ptrs[k] = irs[k];
            if (pinned && irs[k])  // the device staging copy of this set
                ptrs[k] = nullptr;  // filled below once the staging buffers exist
            if (irs[k] && kernel_ok) {
                slot = (slot + 1) % kSlots;
                entries[k] = slot * (int)S;
            }
        }
        if (pinned) {
            const long need_x = S * Kp * period * L, need_ir = Kp * S * std::max<long>(ir_length, 1);
            if (e->swh_cap_x < need_x || e->swh_cap_ir < need_ir) {
                CK(cudaDeviceSynchronize());
                for (int b = 0; b < 2; ++b) {
                    if (e->swh_x[b]) CK(cudaFree(e->swh_x[b]));
                    if (e->swh_y[b]) CK(cudaFree(e->swh_y[b]));
                    if (e->swh_ir[b]) CK(cudaFree(e->swh_ir[b]));
                    e->swh_x[b] = dalloc<float>(need_x);
                    e->swh_y[b] = dalloc<float>(need_x);
                    e->swh_ir[b] = dalloc<float>(need_ir);
                }
                e->swh_cap_x = need_x;
                e->swh_cap_ir = need_ir;
            }
            for (long k = 0; k < nsw; ++k)
                if (irs[k]) ptrs[k] = e->swh_ir[(k / Kp) & 1] + (k % Kp) * S * ir_length;
        }
        if (kernel_ok && e->sw_cap < nsw) {
            CK(cudaStreamSynchronize(e->stream));
            if (e->d_sw_irs) CK(cudaFree(e->d_sw_irs));
            if (e->d_sw_entry) CK(cudaFree(e->d_sw_entry));
            e->d_sw_irs = dalloc<const float*>(nsw);
            e->d_sw_entry = dalloc<int>(nsw);
            e->sw_cap = nsw;
        }
        if (kernel_ok) {  // stream-ordered behind any earlier switching launch still reading the tables
            CK(cudaMemcpyAsync(e->d_sw_irs, ptrs.data(), sizeof(const float*) * nsw, cudaMemcpyHostToDevice,
                               e->stream));
            CK(cudaMemcpyAsync(e->d_sw_entry, entries.data(), sizeof(int) * nsw, cudaMemcpyHostToDevice, e->stream));
            CK(cudaStreamSynchronize(e->stream));  // host tables may go away when we return
        }
        auto launch = [&](long k0, long nk, long hops, const float* din, long din_stride, float* dout, long dout_stride) {
            e->sw_irs_launch = e->d_sw_irs + k0;
            e->sw_entry_launch = e->d_sw_entry + k0;
            e->sw_count_launch = (int)nk;
            e->sw_period_launch = (int)period;
            e->sw_len_launch = ir_length;
            try {
                launch_hops(e, e->hops, hops, din, din_stride, dout, dout_stride, nullptr, 0);
            } catch (...) {
                e->sw_count_launch = 0;
                e->sw_irs_launch = nullptr;
                e->sw_entry_launch = nullptr;
                throw;
            }
            e->sw_count_launch = 0;
            e->sw_irs_launch = nullptr;
            e->sw_entry_launch = nullptr;
            e->hops += hops;
        };
        (void)launch;
        if (!pinned) {
            launch(0, nsw, n_hops, in, in_lane_stride, out, out_lane_stride);
        } else {
            CK(cudaEventRecord(e->ev_start, e->stream));
            CK(cudaStreamWaitEvent(e->h2d, e->ev_start, 0));
            CK(cudaStreamWaitEvent(e->d2h, e->ev_start, 0));
            for (long c = 0, k0 = 0; k0 < nsw; ++c, k0 += Kp) {
                const int b = (int)(c & 1);
                const long nk = std::min(Kp, nsw - k0), h0 = k0 * period;
                const long hops = std::min(nk * period, n_hops - h0), w = Kp * period * L;
                // H2D: the chunk's hops and sets, after the launch that last read buffer b
                if (c >= 2) CK(cudaStreamWaitEvent(e->h2d, e->ev_k[b], 0));
                CK(copy_rows(e->swh_x[b], w * sizeof(float), in + h0 * L, in_lane_stride * sizeof(float),
                                     hops * L * sizeof(float), S, cudaMemcpyHostToDevice, e->h2d));
                // the chunk's sets; runs of sets that are consecutive in host memory (and so in the
                // staging buffer) go as one copy when they lie in one pinned allocation (the
                // runtime rejects a range spanning two: then one copy per set)
                for (long k = k0; k < k0 + nk;) {
                    if (!irs[k]) {
                        ++k;
                        continue;
                    }
                    long k2 = k + 1;
                    while (e->pipe_merge && k2 < k0 + nk && irs[k2] && irs[k2] == irs[k2 - 1] + S * ir_length &&
                           ptrs[k2] == ptrs[k2 - 1] + S * ir_length)
                        ++k2;
                    const size_t set_bytes = sizeof(float) * S * ir_length;
                    if (cudaMemcpyAsync(const_cast<float*>(ptrs[k]), irs[k], set_bytes * (k2 - k),
                                        cudaMemcpyHostToDevice, e->h2d) != cudaSuccess) {
                        (void)cudaGetLastError();  // not sticky: an argument error
                        for (long kk = k; kk < k2; ++kk)
                            CK(cudaMemcpyAsync(const_cast<float*>(ptrs[kk]), irs[kk], set_bytes, cudaMemcpyHostToDevice,
                                               e->h2d));
                    }
                    k = k2;
                }
                CK(cudaEventRecord(e->ev_in[b], e->h2d));
                CK(cudaStreamWaitEvent(e->stream, e->ev_in[b], 0));
                if (c >= 2) CK(cudaStreamWaitEvent(e->stream, e->ev_o[b], 0));  // D2H of chunk c-2 done
                if (kernel_ok) {
                    launch(k0, nk, hops, e->swh_x[b], w, e->swh_y[b], w);
                } else {  // the loop on device-resident staging (in-stream K4 launches)
                    for (long k = k0; k < k0 + nk; ++k) {
                        const long r0 = (k - k0) * period, kc = std::min(period, hops - r0);
                        if (irs[k]) {
                            const int rc = tvolap_exchange_filter(e, ptrs[k], ir_length, S);
                            if (rc) throw ApiError{rc, g_err};
                        }
                        process_hops_impl(e, e->swh_x[b] + r0 * L, w, e->swh_y[b] + r0 * L, w, kc, nullptr);
                    }
                }
                CK(cudaEventRecord(e->ev_k[b], e->stream));
                CK(cudaStreamWaitEvent(e->d2h, e->ev_k[b], 0));
                CK(copy_rows(out + h0 * L, out_lane_stride * sizeof(float), e->swh_y[b], w * sizeof(float),
                                     hops * L * sizeof(float), S, cudaMemcpyDeviceToHost, e->d2h));
                CK(cudaEventRecord(e->ev_o[b], e->d2h));
            }
            CK(cudaEventRecord(e->ev_start, e->d2h));  // later work on the engine stream sees the outputs
            CK(cudaStreamWaitEvent(e->stream, e->ev_start, 0));
        }
        if (kernel_ok) {  // (the loop path keeps its own slot rotation and counts)
            e->active = slot;
            for (int i = 0; i < kSlots; ++i) CK(cudaEventRecord(e->ev_slot[i], e->stream));  // every slot touched
            CK(cudaEventRecord(e->ev_main, e->stream));
            e->fwd += (uint64_t)(S * n_hops);
            e->inv += (uint64_t)(S * e->E * n_hops);
            e->macs += (uint64_t)(S * e->E * e->M * n_hops);
        }
        if (pinned && !e->host_async) CK(cudaStreamSynchronize(e->stream));
    });
}

int tvolap_exchange_filter(tvolap_engine* e, const float* ir, long ir_length, long channels) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    if (e->bank) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "exchange_filter on a bank engine; use select_bank");
    if (!ir || ir_length < 1 || channels < 1)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "partition: impulse response is empty");
    if (channels != e->S) return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter channel count differs");
    const long need = (ir_length + 2 * e->L - 1) / (2 * e->L);
    if (need > e->M)
        return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter partition count differs");
    return guarded([&] {
        CK(cudaSetDevice(e->device));
        std::lock_guard<std::mutex> lock(e->mu);
        // A set still being transformed on the side stream into the next slot is superseded
        // (last staged wins): whatever transforms the replacement into the same slot on the
        // engine stream (at latch, or fused into the first hop launch) must come after it.
        if (e->pending && e->staged_on_side) CK(cudaStreamWaitEvent(e->stream, e->ev_side, 0));
        set_release(e->pending_ext);
        e->pending_ext = nullptr;
        // Stage only: the next process call's first kernel transforms the set (K4 fused).
        // Device IRs are used in place; host IRs are uploaded on the side stream into one of
        // two buffers, after the kernel that consumed that buffer last time.
        const size_t count = (size_t)channels * ir_length;
        if (classify(ir) == Mem::Device) {
            e->staged_ir = ir;
            e->staged_buf = -1;
        } else {
            const int b = e->irst_next;
            e->irst_next = (b + 1) % e->ir_stages;
            CK(cudaStreamWaitEvent(e->upl, e->ev_used[b], 0));
            if (e->irst_cap[b] < count) {
                CK(cudaStreamSynchronize(e->upl));
                CK(cudaStreamSynchronize(e->side));
                CK(cudaStreamSynchronize(e->stream));
                if (e->d_irst[b]) CK(cudaFree(e->d_irst[b]));
                e->d_irst[b] = dalloc<float>(count);
                e->irst_cap[b] = count;
            }
            CK(cudaMemcpyAsync(e->d_irst[b], ir, count * sizeof(float), cudaMemcpyHostToDevice, e->upl));
            CK(cudaEventRecord(e->ev_up[b], e->upl));
            e->staged_ir = e->d_irst[b];
            e->staged_buf = b;
        }
        e->staged_len = ir_length;
        // device-resident sets: K4 on the engine stream, PDL-chained between hop launches; sets
        // uploaded from the host: K4 on the side stream right behind its upload (a cross-stream
        // wait would break the PDL chain and serialise K4 with the hop kernels)
        e->staged_in_stream = e->k4_stream && e->staged_buf < 0;
        e->staged_on_side = e->k4_side && !e->staged_in_stream;
        if (e->staged_on_side) {  // transform now on the side stream, after the last reader of the target slot
            const int target = (e->active + 1) % kSlots;
            CK(cudaStreamWaitEvent(e->side, e->ev_slot[target], 0));
            if (e->staged_buf >= 0) CK(cudaStreamWaitEvent(e->side, e->ev_up[e->staged_buf], 0));
            CK(tvb::launch_partition((int)e->L, (int)e->M, channels, e->staged_ir, ir_length, ir_length, e->pool,
                                     (long)target * e->S, e->tw, e->pk, e->side));
            ++e->launches;
            CK(cudaEventRecord(e->ev_side, e->side));
            if (e->staged_buf >= 0) CK(cudaEventRecord(e->ev_used[e->staged_buf], e->side));
        }
        e->pending = true;  // last staged filter wins (engine.cpp:47)
    });
}

int tvolap_select_bank(tvolap_engine* e, const int32_t* idx) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    if (!e->bank) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "select_bank on a filter-set engine");
    if (!idx) return set_err(TVOLAP_ERR_INVALID_INPUT, "null selection");
    for (long s = 0; s < e->S; ++s)
        if (idx[s] < 0 || idx[s] >= e->n_bank) return set_err(TVOLAP_ERR_INVALID_INPUT, "bank index out of range");
    std::lock_guard<std::mutex> lock(e->mu);
    e->staged.assign(idx, idx + e->S);
    e->sel_staged = true;
    return TVOLAP_OK;
}

int tvolap_reset(tvolap_engine* e) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    return guarded([&] {
        CK(cudaSetDevice(e->device));
        CK(cudaMemsetAsync(e->ring, 0, (size_t)e->S * 2 * e->D * e->N * sizeof(float2), e->stream));
        CK(cudaMemsetAsync(e->hist, 0, (size_t)e->S * e->L * sizeof(float), e->stream));
        CK(cudaMemsetAsync(e->ola, 0, (size_t)e->S * e->E * 3 * e->L * sizeof(float), e->stream));
        e->hops = 0;  // staged filters / selections stay staged (test_engine.cpp:218-232)
    });
}

long tvolap_hop(const tvolap_engine* e) { return e ? e->L : 0; }
long tvolap_channels(const tvolap_engine* e) { return e ? e->S : 0; }
long tvolap_output_channels(const tvolap_engine* e) { return e ? e->S * e->E : 0; }
long tvolap_partition_count(const tvolap_engine* e) { return e ? e->M : 0; }
long tvolap_delay_line_depth(const tvolap_engine* e) { return e ? 2 * e->M - 1 : 0; }
long tvolap_latency(const tvolap_engine* e) { return e ? 2 * e->L : 0; }
long tvolap_switching_latency(const tvolap_engine* e) { return e ? e->L : 0; }
long tvolap_stream_delay(const tvolap_engine* e) { return e ? e->L : 0; }
long tvolap_hops_processed(const tvolap_engine* e) { return e ? e->hops : 0; }

int tvolap_op_counts(const tvolap_engine* e, uint64_t* forward, uint64_t* inverse, uint64_t* macs) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    if (forward) *forward = e->fwd;
    if (inverse) *inverse = e->inv;
    if (macs) *macs = e->macs;
    return TVOLAP_OK;
}

int tvolap_set_stream(tvolap_engine* e, void* stream) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    return guarded([&] {
        CK(cudaSetDevice(e->device));
        cudaStream_t next = stream ? static_cast<cudaStream_t>(stream) : e->own;
        if (next == e->stream) return;
        CK(cudaEventRecord(e->ev_start, e->stream));  // keep order across the switch
        CK(cudaStreamWaitEvent(next, e->ev_start, 0));
        e->stream = next;
    });
}

int tvolap_set_profiling(tvolap_engine* e, int enable) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    e->profiling = enable != 0;
    e->prof_used = 0;
    return TVOLAP_OK;
}

int tvolap_kernel_time(tvolap_engine* e, double* total_ms, long* launches) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    return guarded([&] {
        CK(cudaSetDevice(e->device));
        double sum = 0.0;
        for (size_t i = 0; i < e->prof_used; ++i) {
            CK(cudaEventSynchronize(e->prof_events[i].second));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e->prof_events[i].first, e->prof_events[i].second));
            sum += ms;
        }
        if (total_ms) *total_ms = sum;
        if (launches) *launches = (long)e->prof_used;
        e->prof_used = 0;
    });
}

int tvolap_set_host_async(tvolap_engine* e, int enable) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    e->host_async = enable != 0;
    return TVOLAP_OK;
}

int tvolap_synchronize(tvolap_engine* e) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    return guarded([&] {
        CK(cudaSetDevice(e->device));
        CK(cudaStreamSynchronize(e->stream));
        CK(cudaStreamSynchronize(e->side));
        CK(cudaGetLastError());
    });
}

int tvolap_launch_config(const tvolap_engine* e, int* ctas_per_source, int* threads_per_cta) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    if (ctas_per_source) *ctas_per_source = e->PB;
    if (threads_per_cta) *threads_per_cta = hop_threads(e);  // what the one-hop launch really uses
    return TVOLAP_OK;
}

int tvolap_set_launch_config(tvolap_engine* e, int ctas_per_source, int threads_per_cta) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    return guarded([&] {
        const int P = ctas_per_source > 0 ? ctas_per_source : e->P;
        const int NT = threads_per_cta > 0 ? threads_per_cta : e->NT;
        validate_launch(e, P, NT);
        e->P = P;
        e->NT = NT;
        if (threads_per_cta > 0) e->fix_nt = NT;  // the one-hop launch honours it (hop_threads)
        if (ctas_per_source > 0) {
            e->PB = P;
            e->geometry_fixed = true;
        }
        pick_block_geometry(e);
    });
}

int tvolap_set_block_config(tvolap_engine* e, int hops_per_block, long block_min) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    return guarded([&] {
        if (hops_per_block != 0) {
            if (hops_per_block != 2 && hops_per_block != 4 && hops_per_block != 8 && hops_per_block != 16)
                throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "hops per block must be 2, 4, 8 or 16"};
            const int jh = hops_per_block / 2;
            if (tvb::block_kernel_smem_bytes((int)e->L, e->PB, (int)e->E, jh, e->bank, e->NTB) > 227 * 1024)
                throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "hop block does not fit in shared memory"};
            e->JH = jh;
            e->geometry_fixed = true;
            pick_block_geometry(e);  // threads / partition groups follow the new block length
        }
        if (block_min > 0) e->block_min = block_min;
    });
}

int tvolap_block_config(const tvolap_engine* e, int* hops_per_block, long* block_min, int* partition_groups) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    if (hops_per_block) *hops_per_block = 2 * e->JH;
    if (block_min) *block_min = e->block_min;
    if (partition_groups) *partition_groups = e->QB;
    return TVOLAP_OK;
}

uint64_t tvolap_kernel_launches(const tvolap_engine* e) { return e ? e->launches : 0; }

uint64_t tvolap_wide_passes(const tvolap_engine* e) { return e ? e->wide_passes : 0; }
uint64_t tvolap_ring_launches(const tvolap_engine* e) { return e ? e->ring_launches : 0; }

// ------------------------------------------------------------------ tuning knobs
// Every A/B switch of the kernel, geometry and pipeline choices is a named knob; the defaults are
// the measured-best choices. Nothing in the library reads the environment.
extern "C++" {
namespace {
struct Knob {
    const char* key;
    long tvolap_engine::*field;  // per-engine knob, or
    long* global;                // process-wide launch knob
    long lo, hi;
    int apply;                   // 0: value only, 1: re-derive launch + block geometry
};
const Knob kKnobs[] = {
    {"block_min", &tvolap_engine::block_min, nullptr, 1, 1L << 40, 0},
    {"k4_side", &tvolap_engine::k4_side, nullptr, 0, 1, 0},
    {"k4_stream", &tvolap_engine::k4_stream, nullptr, 0, 1, 0},
    {"ir_stages", &tvolap_engine::ir_stages, nullptr, 1, kIrStage, 0},
    {"wide", &tvolap_engine::wide_mode, nullptr, 0, 2, 0},
    {"wide_warp_fft", &tvolap_engine::wide_warp_fft, nullptr, 0, 1, 0},
    {"wide_q", &tvolap_engine::wide_q, nullptr, -1, 64, 0},
    {"wide_stage", &tvolap_engine::wide_stage, nullptr, 0, 1, 0},
    {"wide_pool_mb", &tvolap_engine::wide_pool_mb, nullptr, 1, 1L << 20, 0},
    {"wide_fuse", &tvolap_engine::wide_fuse, nullptr, 0, 1, 0},
    {"wide_xe_mb", &tvolap_engine::wide_xe_mb, nullptr, 1, 1L << 20, 0},
    {"wide_period", &tvolap_engine::wide_period, nullptr, 0, 1, 0},
    {"bank_pass", &tvolap_engine::bank_pass, nullptr, 0, 1, 0},
    {"bank_pass_mb", &tvolap_engine::bank_pass_mb, nullptr, 1, 1L << 20, 0},
    {"bank_pass_hops", &tvolap_engine::bank_pass_hops, nullptr, 0, 1L << 30, 0},
    {"bank_pass_q", &tvolap_engine::bank_pass_q, nullptr, 0, 64, 0},
    {"bank_pass_jh", &tvolap_engine::bank_pass_jh, nullptr, 0, 32, 0},
    {"k1_small", &tvolap_engine::k1_small, nullptr, 0, 1, 0},
    {"hop_ring", &tvolap_engine::hop_ring, nullptr, 0, 4, 0},
    {"zero_copy", &tvolap_engine::zero_copy, nullptr, 0, 1, 0},
    {"bank_pass_tpc", &tvolap_engine::bank_pass_tpc, nullptr, 0, 1L << 20, 0},
    {"entry_order", &tvolap_engine::entry_order, nullptr, 0, 1, 0},
    {"pipe_merge", &tvolap_engine::pipe_merge, nullptr, 0, 1, 0},
    {"pipe_mb", &tvolap_engine::pipe_mb, nullptr, 1, 1L << 20, 0},
    {"pipe_log2", &tvolap_engine::pipe_log2, nullptr, 10, 34, 0},
    {"k4_gap_mult", &tvolap_engine::k4_gap_mult, nullptr, 1, 64, 0},
    {"sw_1024", &tvolap_engine::sw_1024, nullptr, 0, 1, 0},
    {"p", &tvolap_engine::fix_p, nullptr, 0, 8, 1},
    {"nt", &tvolap_engine::fix_nt, nullptr, 0, 1024, 1},
    {"pb", &tvolap_engine::fix_pb, nullptr, 0, 8, 1},
    {"jh", &tvolap_engine::fix_jh, nullptr, 0, 8, 1},
    {"ntb", &tvolap_engine::ntb, nullptr, 32, 256, 1},
    {"pdl", nullptr, &tvb::g_launch_pdl, 0, 1, 0},
    {"k4_warp", nullptr, &tvb::g_launch_k4_warp, 0, 1, 0},
    {"k4_prefetch", nullptr, &tvb::g_launch_k4_prefetch, 0, 1, 0},
};
std::mutex g_tune_mu;
std::vector<std::pair<const Knob*, long>> g_default_tuning;  // engine knobs applied at creation

const Knob& find_knob(const char* key) {
    if (key)
        for (const Knob& k : kKnobs)
            if (std::strcmp(k.key, key) == 0) return k;
    throw ApiError{TVOLAP_ERR_INVALID_INPUT, std::string("unknown tuning key: ") + (key ? key : "(null)")};
}

void check_range(const Knob& k, long v) {
    if (v < k.lo || v > k.hi)
        throw ApiError{TVOLAP_ERR_INVALID_INPUT, std::string("tuning ") + k.key + " must be in [" +
                                                     std::to_string(k.lo) + ", " + std::to_string(k.hi) + "]"};
}

void apply_default_tuning(tvolap_engine* e) {
    std::lock_guard<std::mutex> lock(g_tune_mu);
    for (const auto& kv : g_default_tuning) e->*(kv.first->field) = kv.second;
}
}  // namespace
}  // extern "C++"

int tvolap_set_tuning(tvolap_engine* e, const char* key, long value) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    return guarded([&] {
        const Knob& k = find_knob(key);
        check_range(k, value);
        if (k.global) {
            *k.global = value;
            return;
        }
        if (k.apply) {  // validate the resulting geometry before committing it
            const long old = e->*k.field;
            e->*k.field = value;
            try {
                pick_launch_config(e);
                validate_launch(e, e->P, e->NT);
                pick_block_geometry(e);
            } catch (...) {
                e->*k.field = old;
                pick_launch_config(e);
                pick_block_geometry(e);
                throw;
            }
        } else {
            e->*k.field = value;
        }
    });
}

int tvolap_get_tuning(const tvolap_engine* e, const char* key, long* value) {
    if (!e || !value) return set_err(TVOLAP_ERR_INVALID_INPUT, "null engine or output");
    return guarded([&] {
        const Knob& k = find_knob(key);
        *value = k.global ? *k.global : e->*k.field;
    });
}

int tvolap_set_default_tuning(const char* key, long value) {
    return guarded([&] {
        const Knob& k = find_knob(key);
        check_range(k, value);
        if (k.global) {
            *k.global = value;
            return;
        }
        std::lock_guard<std::mutex> lock(g_tune_mu);
        for (auto& kv : g_default_tuning)
            if (kv.first == &k) {
                kv.second = value;
                return;
            }
        g_default_tuning.emplace_back(&k, value);
    });
}

int tvolap_reset_default_tuning(void) {
    std::lock_guard<std::mutex> lock(g_tune_mu);
    g_default_tuning.clear();
    tvb::g_launch_pdl = tvb::g_launch_k4_warp = tvb::g_launch_k4_prefetch = 1;
    return TVOLAP_OK;
}

const char* tvolap_tuning_keys(void) {
    static const std::string keys = [] {
        std::string out;
        for (const Knob& k : kKnobs) out += (out.empty() ? "" : ",") + std::string(k.key);
        return out;
    }();
    return keys.c_str();
}

// ------------------------------------------------------------------ spectral primitives
namespace {

struct DevBuf {
    void* p = nullptr;
    explicit DevBuf(size_t bytes) { CK(cudaMalloc(&p, std::max<size_t>(bytes, 1))); }
    ~DevBuf() { cudaFree(p); }
};

// Device view of a host-or-device input buffer.
const void* dev_in(const void* src, size_t bytes, std::vector<DevBuf*>& keep) {
    if (classify(src) == Mem::Device) return src;
    auto* b = new DevBuf(bytes);
    keep.push_back(b);
    CK(cudaMemcpy(b->p, src, bytes, cudaMemcpyHostToDevice));
    return b->p;
}

struct Keep {
    std::vector<DevBuf*> v;
    ~Keep() {
        for (auto* b : v) delete b;
    }
};

void copy_out(void* dst, const void* dev, size_t bytes) {
    CK(cudaMemcpy(dst, dev, bytes, classify(dst) == Mem::Device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost));
}

}  // namespace

int tvolap_forward_real(int device, long n, long batch, const float* x, float* bins) {
    if (n < 8 || !is_pow2(n))
        return set_err(TVOLAP_ERR_INVALID_SIZE,
                       "forward_real: block length must be a power of two >= 8, got " + std::to_string(n));
    if (batch < 1 || !x || !bins) return set_err(TVOLAP_ERR_INVALID_INPUT, "empty batch");
    return guarded([&] {
        require_device(device);
        Keep k;
        Tables t(n / 2);
        const float2* tw = (const float2*)dev_in(t.tw.data(), sizeof(float2) * t.tw.size(), k.v);
        const float2* pk = (const float2*)dev_in(t.pk.data(), sizeof(float2) * t.pk.size(), k.v);
        const float* dx = (const float*)dev_in(x, sizeof(float) * n * batch, k.v);
        DevBuf out(sizeof(float2) * (n / 2 + 1) * batch);
        CK(tvb::launch_forward_real(n, batch, dx, (float2*)out.p, tw, pk, nullptr));
        copy_out(bins, out.p, sizeof(float2) * (n / 2 + 1) * batch);
    });
}

int tvolap_inverse_real(int device, long n, long batch, const float* bins, float* x) {
    if (n < 8 || !is_pow2(n))
        return set_err(TVOLAP_ERR_INVALID_SIZE,
                       "inverse_real: transform length must be a power of two >= 8, got " + std::to_string(n));
    if (batch < 1 || !x || !bins) return set_err(TVOLAP_ERR_INVALID_INPUT, "empty batch");
    const long nb = n / 2 + 1;
    return guarded([&] {
        require_device(device);
        std::vector<float> hb;
        const float* hv = bins;
        if (classify(bins) == Mem::Device) {
            hb.resize(2 * nb * batch);
            CK(cudaMemcpy(hb.data(), bins, sizeof(float) * hb.size(), cudaMemcpyDeviceToHost));
            hv = hb.data();
        }
        for (long b = 0; b < batch; ++b)
            if (hv[2 * (b * nb) + 1] != 0.f || hv[2 * (b * nb + nb - 1) + 1] != 0.f)
                throw ApiError{TVOLAP_ERR_INVALID_SPECTRUM,
                               "inverse_real: DC and Nyquist bins must have zero imaginary part"};
        Keep k;
        Tables t(n / 2);
        const float2* tw = (const float2*)dev_in(t.tw.data(), sizeof(float2) * t.tw.size(), k.v);
        const float2* pk = (const float2*)dev_in(t.pk.data(), sizeof(float2) * t.pk.size(), k.v);
        const float2* db = (const float2*)dev_in(bins, sizeof(float2) * nb * batch, k.v);
        DevBuf out(sizeof(float) * n * batch);
        CK(tvb::launch_inverse_real(n, batch, db, (float*)out.p, tw, pk, nullptr));
        copy_out(x, out.p, sizeof(float) * n * batch);
    });
}

int tvolap_mac(int device, long nbins, long batch, const float* acc, const float* a, const float* b, float* out) {
    if (nbins < 1 || batch < 1 || !acc || !a || !b || !out)
        return set_err(TVOLAP_ERR_INVALID_SIZE, "mac: bin counts differ");
    return guarded([&] {
        require_device(device);
        Keep k;
        const size_t bytes = sizeof(float2) * nbins * batch;
        const float2* da = (const float2*)dev_in(acc, bytes, k.v);
        const float2* dx = (const float2*)dev_in(a, bytes, k.v);
        const float2* dy = (const float2*)dev_in(b, bytes, k.v);
        DevBuf o(bytes);
        CK(tvb::launch_mac(nbins, batch, da, dx, dy, (float2*)o.p, nullptr));
        copy_out(out, o.p, bytes);
    });
}

int tvolap_hann_window(long hop, float* w) {
    if (hop < 2)
        return set_err(TVOLAP_ERR_INVALID_SIZE, "hann_window: hop size must be >= 2, got " + std::to_string(hop));
    std::vector<float> v = hann(hop);
    std::memcpy(w, v.data(), sizeof(float) * v.size());
    return TVOLAP_OK;
}

int tvolap_partition(int device, long hop, long channels, long ir_length, const float* ir, long min_partitions,
                     float* spectra, long* partitions) {
    if (ir_length < 1 || channels < 1 || !ir)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "partition: impulse response is empty");
    if (hop < 2 || !is_pow2(4 * hop))
        return set_err(TVOLAP_ERR_INVALID_SIZE, "partition: 4L must be a power of two, got L = " + std::to_string(hop));
    return guarded([&] {
        require_device(device);
        const long N = 2 * hop, slice = 2 * hop;
        const long M = std::max((ir_length + slice - 1) / slice, std::max<long>(min_partitions, 1));
        if (partitions) *partitions = M;
        if (!spectra) return;
        Keep k;
        Tables t(N);
        const float2* tw = (const float2*)dev_in(t.tw.data(), sizeof(float2) * t.tw.size(), k.v);
        const float2* pk = (const float2*)dev_in(t.pk.data(), sizeof(float2) * t.pk.size(), k.v);
        const float* dir = (const float*)dev_in(ir, sizeof(float) * channels * ir_length, k.v);
        DevBuf pool(sizeof(float2) * channels * M * N);
        CK(tvb::launch_partition((int)hop, (int)M, channels, dir, ir_length, ir_length, (float2*)pool.p, 0, tw, pk,
                                 nullptr));
        std::vector<float2> packed((size_t)channels * M * N);
        CK(cudaMemcpy(packed.data(), pool.p, sizeof(float2) * packed.size(), cudaMemcpyDeviceToHost));
        std::vector<float> full((size_t)channels * M * (N + 1) * 2);
        for (long f = 0; f < channels * M; ++f) {
            const float2* src = packed.data() + f * N;
            float* dst = full.data() + f * (N + 1) * 2;
            dst[0] = src[0].x;
            dst[1] = 0.f;
            for (long q = 1; q < N; ++q) {
                dst[2 * q] = src[q].x;
                dst[2 * q + 1] = src[q].y;
            }
            dst[2 * N] = src[0].y;
            dst[2 * N + 1] = 0.f;
        }
        if (classify(spectra) == Mem::Device)
            CK(cudaMemcpy(spectra, full.data(), sizeof(float) * full.size(), cudaMemcpyHostToDevice));
        else
            std::memcpy(spectra, full.data(), sizeof(float) * full.size());
    });
}

int tvolap_gen_white_device(int device, uint64_t seed, long lane0, long lanes, long t0, long n, float* out,
                            long stride) {
    return guarded([&] {
        require_device(device);
        if (classify(out) != Mem::Device) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "output must be device memory"};
        CK(tvb::launch_gen_white(seed, lane0, lanes, t0, n, out, stride, nullptr));
        CK(cudaDeviceSynchronize());
    });
}

int tvolap_gen_irs_device(int device, uint64_t seed, long count, const long* lanes, const long* ears,
                          const long* ks, const double* t60, double fs, long len, float* out) {
    return guarded([&] {
        require_device(device);
        if (classify(out) != Mem::Device) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "output must be device memory"};
        Keep k;
        const long* dl = (const long*)dev_in(lanes, sizeof(long) * count, k.v);
        const long* de = (const long*)dev_in(ears, sizeof(long) * count, k.v);
        const long* dk = (const long*)dev_in(ks, sizeof(long) * count, k.v);
        const double* dt = (const double*)dev_in(t60, sizeof(double) * count, k.v);
        CK(tvb::launch_gen_irs(seed, count, dl, de, dk, dt, fs, len, out, nullptr));
        CK(cudaDeviceSynchronize());
    });
}

int tvolap_mix_device(int device, long sources, long ears, long samples, const float* out, long out_stride,
                      float* mix, long mix_stride, void* stream) {
    return guarded([&] {
        CK(cudaSetDevice(device));
        CK(tvb::launch_mix(sources, ears, samples, out, out_stride, mix, mix_stride, (cudaStream_t)stream));
    });
}

// ---- device-resident filter partition sets (partition.hpp:21-43)
int tvolap_set_create(tvolap_set** out, int device, long hop, long channels, long ir_length, const float* ir,
                      long min_partitions) {
    if (!out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null output handle");
    *out = nullptr;
    if (ir_length < 1 || channels < 1 || !ir)  // partition.cpp:21-24, in the reference's order
        return set_err(TVOLAP_ERR_INVALID_INPUT, "partition: impulse response is empty");
    if (hop < 2 || !is_pow2(4 * hop))
        return set_err(TVOLAP_ERR_INVALID_SIZE, "partition: 4L must be a power of two, got L = " + std::to_string(hop));
    return guarded([&] {
        require_device(device);
        auto* st = new tvolap_set();
        try {
            st->device = device;
            st->L = hop;
            st->N = 2 * hop;
            st->S = channels;
            st->source_length = ir_length;
            st->M = std::max((ir_length + 2 * hop - 1) / (2 * hop), std::max<long>(min_partitions, 1));
            const size_t elems = (size_t)channels * st->M * st->N + (size_t)tvb::kWideTail * st->N;
            st->spec = dalloc<float2>(elems);
            CK(cudaMemset(st->spec, 0, elems * sizeof(float2)));  // (synchronous: done before the K4 below)
            Keep k;
            Tables t(st->N);
            const float2* tw = (const float2*)dev_in(t.tw.data(), sizeof(float2) * t.tw.size(), k.v);
            const float2* pk = (const float2*)dev_in(t.pk.data(), sizeof(float2) * t.pk.size(), k.v);
            const float* dir = (const float*)dev_in(ir, sizeof(float) * channels * ir_length, k.v);
            cudaStream_t sm = nullptr;  // a private stream: no device-wide synchronisation
            CK(cudaStreamCreateWithFlags(&sm, cudaStreamNonBlocking));
            const cudaError_t e1 = tvb::launch_partition((int)hop, (int)st->M, channels, dir, ir_length, ir_length,
                                                         st->spec, 0, tw, pk, sm);
            const cudaError_t e2 = cudaStreamSynchronize(sm);
            cudaStreamDestroy(sm);
            CK(e1);
            CK(e2);
        } catch (...) {
            set_release(st);
            throw;
        }
        *out = st;
    });
}

int tvolap_set_release(tvolap_set* s) {
    set_release(s);
    return TVOLAP_OK;
}

int tvolap_set_geometry(const tvolap_set* s, long* hop, long* partitions, long* channels, long* source_length) {
    if (!s) return set_err(TVOLAP_ERR_INVALID_INPUT, "null set");
    if (hop) *hop = s->L;
    if (partitions) *partitions = s->M;
    if (channels) *channels = s->S;
    if (source_length) *source_length = s->source_length;
    return TVOLAP_OK;
}

// spectra[((c * M + m) * (2L + 1) + k) * 2 + {re, im}], host or device (tvolap_partition's layout)
int tvolap_set_spectra(const tvolap_set* s, float* spectra) {
    if (!s || !spectra) return set_err(TVOLAP_ERR_INVALID_INPUT, "null set or output");
    return guarded([&] {
        CK(cudaSetDevice(s->device));
        const long N = s->N, F = s->S * s->M;
        std::vector<float2> packed((size_t)F * N);
        CK(cudaMemcpy(packed.data(), s->spec, sizeof(float2) * packed.size(), cudaMemcpyDeviceToHost));
        std::vector<float> full((size_t)F * (N + 1) * 2);
        for (long f = 0; f < F; ++f) {
            const float2* src = packed.data() + f * N;
            float* dst = full.data() + f * (N + 1) * 2;
            dst[0] = src[0].x;
            dst[1] = 0.f;
            for (long q = 1; q < N; ++q) {
                dst[2 * q] = src[q].x;
                dst[2 * q + 1] = src[q].y;
            }
            dst[2 * N] = src[0].y;
            dst[2 * N + 1] = 0.f;
        }
        if (classify(spectra) == Mem::Device)
            CK(cudaMemcpy(spectra, full.data(), sizeof(float) * full.size(), cudaMemcpyHostToDevice));
        else
            std::memcpy(spectra, full.data(), sizeof(float) * full.size());
    });
}

// reassemble (partition.cpp:53-65): inverse-transform every partition, keep its first 2L samples,
// concatenate: out[c * (2 L M) + n] (the source response zero-padded to M * 2L taps)
int tvolap_set_reassemble(const tvolap_set* s, float* out) {
    if (!s || !out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null set or output");
    const long n = 4 * s->L, F = s->S * s->M, slice = 2 * s->L;
    std::vector<float> bins((size_t)F * (n / 2 + 1) * 2), y((size_t)F * n);
    if (int rc = tvolap_set_spectra(s, bins.data())) return rc;
    if (int rc = tvolap_inverse_real(s->device, n, F, bins.data(), y.data())) return rc;
    return guarded([&] {
        std::vector<float> res((size_t)F * slice);
        for (long f = 0; f < F; ++f) std::memcpy(res.data() + f * slice, y.data() + f * n, sizeof(float) * slice);
        if (classify(out) == Mem::Device) {
            CK(cudaSetDevice(s->device));
            CK(cudaMemcpy(out, res.data(), sizeof(float) * res.size(), cudaMemcpyHostToDevice));
        } else {
            std::memcpy(out, res.data(), sizeof(float) * res.size());
        }
    });
}

// TvolapEngine(shared_ptr<const FilterPartitionSet>) (engine.hpp:35, engine.cpp:9-32): the engine
// reads the set's spectra in place (no K4 at construction).
int tvolap_create_from_set(tvolap_engine** out, const tvolap_set* s) {
    if (!out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null output handle");
    *out = nullptr;
    if (!s) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "engine requires a filter partition set");
    tvolap_engine* e = nullptr;
    const int rc = guarded([&] {
        require_device(s->device);
        e = new tvolap_engine();
        try {
            init_common(e, s->device, s->L, s->S, 1, s->M);
            const size_t slot = (size_t)s->S * s->M * e->N;
            e->pool = dalloc<float2>(kSlots * slot + (size_t)tvb::kWideTail * e->N);
            CK(cudaMemsetAsync(e->pool, 0, (kSlots * slot + (size_t)tvb::kWideTail * e->N) * sizeof(float2), e->stream));
            set_retain(s);
            e->active_ext = s;
            CK(cudaStreamSynchronize(e->stream));
        } catch (...) {
            delete e;
            e = nullptr;
            throw;
        }
    });
    *out = e;
    return rc;
}

// exchange_filter(shared_ptr<const FilterPartitionSet>) (engine.hpp:55, engine.cpp:37-48): O(1) —
// validate, stage (last wins), latch at the next process call; no transform.
int tvolap_exchange_set(tvolap_engine* e, const tvolap_set* s) {
    if (!e) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null engine");
    if (e->bank) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "exchange_filter on a bank engine; use select_bank");
    if (!s) return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter is null");
    if (s->L != e->L) return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter hop differs");
    if (s->M != e->M) return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter partition count differs");
    if (s->S != e->S) return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter channel count differs");
    if (s->device != e->device)
        return set_err(TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter lives on another device");
    return guarded([&] {
        CK(cudaSetDevice(e->device));
        std::lock_guard<std::mutex> lock(e->mu);
        drop_pending(e);  // last staged filter wins
        set_retain(s);
        e->pending_ext = s;
    });
}

// ---- NCCL (C3's cross-GPU mix), loaded at first use so the library has no link-time dependency
extern "C++" {
namespace {
struct NcclApi {
    bool ok = false;
    std::string err;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static const NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
            return a;
        }
        auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::decay_t<decltype(f)>>(dlsym(h, name)); };
        sym(a.get_unique_id, "ncclGetUniqueId");
        sym(a.comm_init_rank, "ncclCommInitRank");
        sym(a.all_reduce, "ncclAllReduce");
        sym(a.comm_destroy, "ncclCommDestroy");
        sym(a.group_start, "ncclGroupStart");
        sym(a.group_end, "ncclGroupEnd");
        sym(a.error_string, "ncclGetErrorString");
        a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.group_start && a.group_end;
        if (!a.ok) a.err = "libnccl.so.2 lacks a required symbol";
        return a;
    }();
    if (!api.ok) throw ApiError{TVOLAP_ERR_CUDA, "NCCL unavailable: " + api.err};
    return api;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const NcclApi& a = nccl();
        throw ApiError{TVOLAP_ERR_CUDA, std::string(what) + ": " + (a.error_string ? a.error_string(r) : "NCCL error")};
    }
}
}  // namespace
}  // extern "C++"

int tvolap_mix_allreduce(int device, long sources, long ears, long samples, const float* out, long out_stride,
                         float* mix, long mix_stride, void* nccl_comm, void* stream) {
    if (!out || !mix || sources < 1 || ears < 1 || samples < 1 || mix_stride < samples || out_stride < samples)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "mix: bad buffers or sizes");
    return guarded([&] {
        CK(cudaSetDevice(device));
        const cudaStream_t st = (cudaStream_t)stream;
        CK(tvb::launch_mix(sources, ears, samples, out, out_stride, mix, mix_stride, st));
        if (!nccl_comm) return;
        const NcclApi& a = nccl();
        auto comm = static_cast<ncclComm_t>(nccl_comm);
        if (mix_stride == samples) {
            nccl_check(a.all_reduce(mix, mix, (size_t)ears * samples, ncclFloat32, ncclSum, comm, st), "ncclAllReduce");
        } else {
            nccl_check(a.group_start(), "ncclGroupStart");
            for (long e2 = 0; e2 < ears; ++e2)
                nccl_check(a.all_reduce(mix + e2 * mix_stride, mix + e2 * mix_stride, (size_t)samples, ncclFloat32,
                                        ncclSum, comm, st),
                           "ncclAllReduce");
            nccl_check(a.group_end(), "ncclGroupEnd");
        }
    });
}

int tvolap_nccl_unique_id(char id_out[128]) {
    if (!id_out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null id buffer");
    return guarded([&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
        ncclUniqueId id;
        nccl_check(nccl().get_unique_id(&id), "ncclGetUniqueId");
        std::memcpy(id_out, &id, sizeof id);
    });
}

int tvolap_nccl_comm_init(void** comm_out, int device, int nranks, int rank, const char id[128]) {
    if (!comm_out || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "nccl comm: bad arguments");
    *comm_out = nullptr;
    return guarded([&] {
        CK(cudaSetDevice(device));
        ncclUniqueId uid;
        std::memcpy(&uid, id, sizeof uid);
        ncclComm_t c = nullptr;
        nccl_check(nccl().comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
        *comm_out = c;
    });
}

int tvolap_nccl_comm_destroy(void* comm) {
    if (!comm) return TVOLAP_OK;
    return guarded([&] { nccl_check(nccl().comm_destroy(static_cast<ncclComm_t>(comm)), "ncclCommDestroy"); });
}

// ======================================================================= peer-memory mix (C3)
struct tvolap_mix_group {
    int device = 0, world = 1, rank = 0;
    long ears = 0, cap = 0;
    float* gather = nullptr;               // this rank's [world][ears][cap] slots
    std::vector<float*> peer;              // every rank's gather buffer in this process's address space
    std::vector<bool> opened;              // peer[r] came from cudaIpcOpenMemHandle
    float** d_slots = nullptr;             // device copy of peer[]
    bool ready = false;
};

int tvolap_mix_group_create(tvolap_mix_group** out, int device, int world, int rank, long ears, long capacity,
                            char ipc_handle_out[64]) {
    if (!out || world < 1 || rank < 0 || rank >= world || ears < 1 || capacity < 1)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "mix group: bad arguments");
    *out = nullptr;
    return guarded([&] {
        require_device(device);
        auto g = std::make_unique<tvolap_mix_group>();
        g->device = device;
        g->world = world;
        g->rank = rank;
        g->ears = ears;
        g->cap = capacity;
        g->gather = dalloc<float>((size_t)world * ears * capacity);
        g->peer.assign(world, nullptr);
        g->opened.assign(world, false);
        g->peer[rank] = g->gather;
        g->d_slots = dalloc<float*>((size_t)world);
        if (ipc_handle_out) {
            static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t is 64 bytes");
            cudaIpcMemHandle_t hnd;
            CK(cudaIpcGetMemHandle(&hnd, g->gather));
            std::memcpy(ipc_handle_out, &hnd, sizeof hnd);
        }
        if (world == 1) {
            CK(cudaMemcpy(g->d_slots, g->peer.data(), sizeof(float*), cudaMemcpyHostToDevice));
            g->ready = true;
        }
        *out = g.release();
    });
}

int tvolap_mix_group_open(tvolap_mix_group* g, const char* handles) {
    if (!g || (!handles && g->world > 1)) return set_err(TVOLAP_ERR_INVALID_INPUT, "mix group: null handles");
    return guarded([&] {
        CK(cudaSetDevice(g->device));
        for (int r = 0; r < g->world; ++r) {
            if (r == g->rank || g->opened[r]) continue;
            cudaIpcMemHandle_t hnd;
            std::memcpy(&hnd, handles + 64 * (size_t)r, sizeof hnd);
            void* p = nullptr;
            CK(cudaIpcOpenMemHandle(&p, hnd, cudaIpcMemLazyEnablePeerAccess));  // NVLink P2P when on another GPU
            g->peer[r] = static_cast<float*>(p);
            g->opened[r] = true;
        }
        CK(cudaMemcpy(g->d_slots, g->peer.data(), sizeof(float*) * g->world, cudaMemcpyHostToDevice));
        g->ready = true;
    });
}

int tvolap_mix_scatter(tvolap_mix_group* g, long sources, long samples, const float* out, long out_stride,
                       void* stream) {
    if (!g || !out || sources < 1 || samples < 1 || out_stride < samples)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "mix scatter: bad buffers or sizes");
    if (samples > g->cap) return set_err(TVOLAP_ERR_INVALID_SIZE, "mix scatter: more samples than the group holds");
    if (!g->ready) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "mix scatter: peer handles not opened");
    return guarded([&] {
        CK(cudaSetDevice(g->device));
        CK(tvb::launch_mix_scatter(sources, g->ears, samples, out, out_stride, g->d_slots, g->world, g->rank, g->cap,
                                   (cudaStream_t)stream));
    });
}

int tvolap_mix_gather(tvolap_mix_group* g, long samples, float* mix, long mix_stride, void* stream) {
    if (!g || !mix || samples < 1 || mix_stride < samples)
        return set_err(TVOLAP_ERR_INVALID_INPUT, "mix gather: bad buffers or sizes");
    if (samples > g->cap) return set_err(TVOLAP_ERR_INVALID_SIZE, "mix gather: more samples than the group holds");
    return guarded([&] {
        CK(cudaSetDevice(g->device));
        CK(tvb::launch_mix_gather(g->ears, samples, g->gather, g->world, g->cap, mix, mix_stride,
                                  (cudaStream_t)stream));
    });
}

int tvolap_mix_group_destroy(tvolap_mix_group* g) {
    if (!g) return TVOLAP_OK;
    return guarded([&] {
        std::unique_ptr<tvolap_mix_group> own(g);
        CK(cudaSetDevice(g->device));
        CK(cudaDeviceSynchronize());
        for (int r = 0; r < g->world; ++r)
            if (g->opened[r]) CK(cudaIpcCloseMemHandle(g->peer[r]));
        CK(cudaFree(g->d_slots));
        CK(cudaFree(g->gather));
    });
}

// ======================================================================= comparison convolvers
// the reference's OLA / OLS / WOLA / TDC / CF-TDC processors
// (reference.cpp:34-320) on the GPU. Host state mirrors the reference classes; the arithmetic
// runs in tvb::launch_fbconv (block FFT forms, the TVOLAP FFT/MAC building blocks with M = 1)
// and tvb::launch_fir (direct forms).
struct tvolap_cmp {
    int device = 0, kind = 0;
    long taps = 0, channels = 0, hop = 0, block = 0;
    cudaStream_t stream = nullptr;
    // direct forms: coefficient sets [C][taps], history [C][taps-1], fade clock (reference.cpp:97-172)
    float *coeffs = nullptr, *old_coeffs = nullptr, *pend_coeffs = nullptr, *history = nullptr, *xx = nullptr;
    long xx_cap = 0;
    bool pending = false;
    long fade_duration = 1, pending_duration = 1, fade_remaining = 0, fade_elapsed = 0;
    int fade_shape = 0, pending_shape = 0;
    // block forms: packed filter spectra [C][B] (active / staged), carried state, scratch frames
    float2 *spec = nullptr, *spec_pend = nullptr, *tw = nullptr, *pk = nullptr;
    bool spec_staged = false;
    float *win = nullptr, *prev = nullptr, *rem = nullptr, *yhat = nullptr;
    long yhat_cap = 0;
    // staging for host buffers
    float *d_in = nullptr, *d_out = nullptr;
    long io_cap = 0;
};

namespace {

void cmp_free(tvolap_cmp* p) {
    for (void* q : {(void*)p->coeffs, (void*)p->old_coeffs, (void*)p->pend_coeffs, (void*)p->history, (void*)p->xx,
                    (void*)p->spec, (void*)p->spec_pend, (void*)p->tw, (void*)p->pk, (void*)p->win, (void*)p->prev,
                    (void*)p->rem, (void*)p->yhat, (void*)p->d_in, (void*)p->d_out})
        if (q) cudaFree(q);
    if (p->stream) cudaStreamDestroy(p->stream);
    delete p;
}

// channel-major IR (stride ir_stride) -> dense device [C][taps]
void cmp_upload(tvolap_cmp* p, float* dst, const float* ir, long ir_stride) {
    const cudaMemcpyKind k = classify(ir) == Mem::Device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpy2DAsync(dst, sizeof(float) * p->taps, ir, sizeof(float) * ir_stride, sizeof(float) * p->taps,
                         p->channels, k, p->stream));
}

// block_filter_spectra (reference.cpp:44-55): IR zero-padded to 2B, real 2B FFT, packed bins —
// the K4 partition transform with hop B/2 and one partition.
void cmp_spectra(tvolap_cmp* p, float2* dst, const float* ir, long ir_stride) {
    const float* src = ir;
    DevBuf* tmp = nullptr;
    if (classify(ir) != Mem::Device) {
        tmp = new DevBuf(sizeof(float) * p->taps * p->channels);
        CK(cudaMemcpy2DAsync(tmp->p, sizeof(float) * p->taps, ir, sizeof(float) * ir_stride, sizeof(float) * p->taps,
                             p->channels, cudaMemcpyHostToDevice, p->stream));
        src = (const float*)tmp->p;
        ir_stride = p->taps;
    }
    const cudaError_t err = tvb::launch_partition((int)(p->block / 2), 1, p->channels, src, ir_stride, p->taps, dst, 0,
                                                  p->tw, p->pk, p->stream);
    if (tmp) {
        cudaStreamSynchronize(p->stream);
        delete tmp;
    }
    CK(err);
}

void cmp_check_filter(const tvolap_cmp* p, const float* ir, long taps, long channels, long ir_stride) {
    if (!ir) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "null impulse response"};
    if (taps != p->taps || channels != p->channels)
        throw ApiError{TVOLAP_ERR_INCOMPATIBLE_FILTER, "replacement filter shape differs"};
    if (ir_stride < taps) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "IR channel stride shorter than the response"};
}

}  // namespace

int tvolap_cmp_create(tvolap_cmp** out, int device, int kind, long taps, long channels, const float* ir,
                      long ir_stride, long hop, long fade_duration, int fade_shape) {
    if (!out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null output handle");
    *out = nullptr;
    tvolap_cmp* p = new tvolap_cmp;
    const int rc = guarded([&] {
        const bool direct = kind == TVOLAP_CMP_TDC || kind == TVOLAP_CMP_CF_TDC;
        const bool block = kind == TVOLAP_CMP_OLA || kind == TVOLAP_CMP_OLS || kind == TVOLAP_CMP_WOLA;
        if (!direct && !block) throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "unknown algorithm"};
        if (direct && hop < 1) throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "hop must be positive"};
        if (direct && (taps < 1 || channels < 1)) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "empty impulse response"};
        if (kind == TVOLAP_CMP_CF_TDC && fade_duration < 1)
            throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "crossfade duration must be >= 1"};
        if (block && (taps < 4 || !is_pow2(taps)))
            throw ApiError{TVOLAP_ERR_INVALID_SIZE,
                           "block fast convolution needs a power-of-two response length >= 4"};
        if (block && taps > 4096)  // one real 2B transform per CTA in shared memory
            throw ApiError{TVOLAP_ERR_INVALID_SIZE, "GPU block convolvers support responses up to 4096 taps"};
        if (block && channels < 1) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "empty impulse response"};
        if (!ir) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "null impulse response"};
        if (ir_stride < taps) throw ApiError{TVOLAP_ERR_INVALID_INPUT, "IR channel stride shorter than the response"};
        require_device(device);
        CK(cudaSetDevice(device));
        p->device = device;
        p->kind = kind;
        p->taps = taps;
        p->channels = channels;
        CK(cudaStreamCreateWithFlags(&p->stream, cudaStreamNonBlocking));
        if (direct) {
            p->hop = hop;
            p->fade_duration = fade_duration;
            p->fade_shape = fade_shape;
            p->coeffs = dalloc<float>(taps * channels);
            p->old_coeffs = dalloc<float>(taps * channels);
            p->pend_coeffs = dalloc<float>(taps * channels);
            p->history = dalloc<float>(std::max<long>(1, (taps - 1) * channels));
            CK(cudaMemsetAsync(p->old_coeffs, 0, sizeof(float) * taps * channels, p->stream));
            CK(cudaMemsetAsync(p->history, 0, sizeof(float) * std::max<long>(1, (taps - 1) * channels), p->stream));
            cmp_upload(p, p->coeffs, ir, ir_stride);
        } else {
            p->block = taps;
            p->hop = kind == TVOLAP_CMP_WOLA ? taps / 2 : taps;
            Tables t(taps);
            p->tw = dalloc<float2>(t.tw.size());
            p->pk = dalloc<float2>(t.pk.size());
            CK(cudaMemcpy(p->tw, t.tw.data(), sizeof(float2) * t.tw.size(), cudaMemcpyHostToDevice));
            CK(cudaMemcpy(p->pk, t.pk.data(), sizeof(float2) * t.pk.size(), cudaMemcpyHostToDevice));
            p->spec = dalloc<float2>(taps * channels);
            p->spec_pend = dalloc<float2>(taps * channels);
            const long rem_len = (kind == TVOLAP_CMP_WOLA ? 3 * p->hop : taps) * channels;
            p->rem = dalloc<float>(rem_len);
            p->prev = dalloc<float>(p->hop * channels);
            CK(cudaMemsetAsync(p->rem, 0, sizeof(float) * rem_len, p->stream));
            CK(cudaMemsetAsync(p->prev, 0, sizeof(float) * p->hop * channels, p->stream));
            std::vector<float> w(taps);  // sqrt(hann_window(B/2)) (reference.cpp:262)
            const double pi = 3.14159265358979323846264338327950288;
            for (long i = 0; i < taps; ++i) w[i] = (float)std::sqrt(1.0 - std::cos(2.0 * pi * (double)i / (double)taps));
            p->win = dalloc<float>(taps);
            CK(cudaMemcpy(p->win, w.data(), sizeof(float) * taps, cudaMemcpyHostToDevice));
            cmp_spectra(p, p->spec, ir, ir_stride);
        }
        CK(cudaStreamSynchronize(p->stream));
    });
    if (rc != TVOLAP_OK) {
        cmp_free(p);
        return rc;
    }
    *out = p;
    return TVOLAP_OK;
}

int tvolap_cmp_destroy(tvolap_cmp* p) {
    if (!p) return TVOLAP_OK;
    cudaSetDevice(p->device);
    cudaStreamSynchronize(p->stream);
    cmp_free(p);
    return TVOLAP_OK;
}

int tvolap_cmp_process_hops(tvolap_cmp* p, const float* in, long in_stride, float* out, long out_stride,
                            long n_hops) {
    if (!p) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null processor");
    if (n_hops < 1) return set_err(TVOLAP_ERR_INVALID_SIZE, "process() expects at least one hop of input");
    if (!in || !out) return set_err(TVOLAP_ERR_INVALID_INPUT, "null input or output");
    const long T = n_hops * p->hop;
    if (in_stride < T || out_stride < T) return set_err(TVOLAP_ERR_INVALID_SIZE, "lane stride shorter than the call");
    return guarded([&] {
        CK(cudaSetDevice(p->device));
        const long C = p->channels;
        // device views of the input / output lanes
        const Mem min = classify(in), mout = classify(out);
        if ((min != Mem::Device || mout != Mem::Device) && p->io_cap < C * T) {
            if (p->d_in) CK(cudaFree(p->d_in));
            if (p->d_out) CK(cudaFree(p->d_out));
            p->d_in = dalloc<float>(C * T);
            p->d_out = dalloc<float>(C * T);
            p->io_cap = C * T;
        }
        const float* din = in;
        long din_stride = in_stride;
        if (min != Mem::Device) {
            CK(cudaMemcpy2DAsync(p->d_in, sizeof(float) * T, in, sizeof(float) * in_stride, sizeof(float) * T, C,
                                 cudaMemcpyHostToDevice, p->stream));
            din = p->d_in;
            din_stride = T;
        }
        float* dout = mout == Mem::Device ? out : p->d_out;
        const long dout_stride = mout == Mem::Device ? out_stride : T;
        if (p->kind == TVOLAP_CMP_TDC || p->kind == TVOLAP_CMP_CF_TDC) {
            if (p->pending) {  // reference.cpp:72-76 / 137-146: latch at the hop boundary
                if (p->kind == TVOLAP_CMP_CF_TDC) {
                    std::swap(p->old_coeffs, p->coeffs);
                    p->fade_duration = p->pending_duration;
                    p->fade_shape = p->pending_shape;
                    p->fade_remaining = p->fade_duration;
                    p->fade_elapsed = 0;
                }
                std::swap(p->coeffs, p->pend_coeffs);
                p->pending = false;
            }
            const long th = p->taps - 1, span = th + T;
            if (p->xx_cap < C * span) {
                if (p->xx) CK(cudaFree(p->xx));
                p->xx = dalloc<float>(C * span);
                p->xx_cap = C * span;
            }
            if (th > 0)
                CK(cudaMemcpy2DAsync(p->xx, sizeof(float) * span, p->history, sizeof(float) * th, sizeof(float) * th, C,
                                     cudaMemcpyDeviceToDevice, p->stream));
            CK(cudaMemcpy2DAsync(p->xx + th, sizeof(float) * span, din, sizeof(float) * din_stride, sizeof(float) * T, C,
                                 cudaMemcpyDeviceToDevice, p->stream));
            const long fade_len = p->kind == TVOLAP_CMP_CF_TDC ? std::min(p->fade_remaining, T) : 0;
            CK(tvb::launch_fir((int)p->taps, C, T, p->xx, span, p->coeffs, p->old_coeffs, dout, dout_stride, fade_len,
                               p->fade_elapsed, p->fade_duration, p->fade_shape, p->stream));
            p->fade_elapsed += fade_len;
            p->fade_remaining -= fade_len;
            if (th > 0)
                CK(cudaMemcpy2DAsync(p->history, sizeof(float) * th, p->xx + T, sizeof(float) * span, sizeof(float) * th,
                                     C, cudaMemcpyDeviceToDevice, p->stream));
        } else {
            if (p->spec_staged) {  // the carried tails keep whatever filter produced them
                std::swap(p->spec, p->spec_pend);
                p->spec_staged = false;
            }
            const long need = C * n_hops * 2 * p->block;
            if (p->yhat_cap < need) {
                if (p->yhat) CK(cudaFree(p->yhat));
                p->yhat = dalloc<float>(need);
                p->yhat_cap = need;
            }
            CK(tvb::launch_fbconv(p->kind, (int)p->block, C, n_hops, din, din_stride, p->prev, p->spec, p->win, p->tw,
                                  p->pk, p->yhat, dout, dout_stride, p->rem, p->stream));
        }
        if (mout != Mem::Device)
            CK(cudaMemcpy2DAsync(out, sizeof(float) * out_stride, dout, sizeof(float) * T, sizeof(float) * T, C,
                                 cudaMemcpyDeviceToHost, p->stream));
        CK(cudaStreamSynchronize(p->stream));
    });
}

int tvolap_cmp_set_filter(tvolap_cmp* p, const float* ir, long taps, long channels, long ir_stride) {
    if (!p) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null processor");
    if (p->kind == TVOLAP_CMP_CF_TDC)  // reference.cpp:134-136: switch with the configured fade
        return tvolap_cmp_switch_filter(p, ir, taps, channels, ir_stride, p->fade_duration, p->fade_shape);
    return guarded([&] {
        cmp_check_filter(p, ir, taps, channels, ir_stride);
        CK(cudaSetDevice(p->device));
        if (p->kind == TVOLAP_CMP_TDC) {
            cmp_upload(p, p->pend_coeffs, ir, ir_stride);
            p->pending = true;
        } else {
            cmp_spectra(p, p->spec_pend, ir, ir_stride);
            p->spec_staged = true;
        }
        CK(cudaStreamSynchronize(p->stream));
    });
}

int tvolap_cmp_switch_filter(tvolap_cmp* p, const float* ir, long taps, long channels, long ir_stride,
                             long fade_duration, int fade_shape) {
    if (!p) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null processor");
    return guarded([&] {
        if (p->kind != TVOLAP_CMP_CF_TDC)
            throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "switch_filter needs a cf-tdc processor"};
        if (p->fade_remaining > 0 || p->pending)
            throw ApiError{TVOLAP_ERR_SWITCH_IN_PROGRESS, "a crossfade is already in progress"};
        cmp_check_filter(p, ir, taps, channels, ir_stride);
        if (fade_duration < 1) throw ApiError{TVOLAP_ERR_INVALID_CONFIGURATION, "crossfade duration must be >= 1"};
        CK(cudaSetDevice(p->device));
        cmp_upload(p, p->pend_coeffs, ir, ir_stride);
        p->pending_duration = fade_duration;
        p->pending_shape = fade_shape;
        p->pending = true;
        CK(cudaStreamSynchronize(p->stream));
    });
}

int tvolap_cmp_reset(tvolap_cmp* p) {
    if (!p) return set_err(TVOLAP_ERR_INVALID_CONFIGURATION, "null processor");
    return guarded([&] {
        CK(cudaSetDevice(p->device));
        const long C = p->channels;
        if (p->history) CK(cudaMemsetAsync(p->history, 0, sizeof(float) * std::max<long>(1, (p->taps - 1) * C), p->stream));
        if (p->rem)
            CK(cudaMemsetAsync(p->rem, 0, sizeof(float) * (p->kind == TVOLAP_CMP_WOLA ? 3 * p->hop : p->taps) * C,
                               p->stream));
        if (p->prev) CK(cudaMemsetAsync(p->prev, 0, sizeof(float) * p->hop * C, p->stream));
        p->fade_remaining = 0;
        p->fade_elapsed = 0;
        CK(cudaStreamSynchronize(p->stream));
    });
}

int tvolap_cmp_geometry(const tvolap_cmp* p, long* out6) {
    if (!p || !out6) return set_err(TVOLAP_ERR_INVALID_INPUT, "null processor or output");
    const bool block = p->block > 0;
    out6[0] = p->hop;
    out6[1] = p->channels;
    out6[2] = block ? p->block : 0;
    out6[3] = p->kind == TVOLAP_CMP_WOLA ? p->block / 2 : 0;
    out6[4] = p->kind == TVOLAP_CMP_CF_TDC ? p->fade_duration : (p->kind == TVOLAP_CMP_WOLA ? p->block / 2 : 0);
    out6[5] = p->fade_remaining > 0 ? 1 : 0;
    return TVOLAP_OK;
}

}  // extern "C"
