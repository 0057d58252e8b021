/*
 * tvolap_b200.h — C-ABI drop-in boundary of the B200-native TVOLAP engine.
 *
 * Replaces the reference's per-hop streaming path:
 *   tvolap::partition(ir, hop, min_partitions)      proj/include/tvolap/partition.hpp:38
 *   tvolap::TvolapEngine ctor                       proj/include/tvolap/engine.hpp:35-36
 *   TvolapEngine::process(input)                    proj/include/tvolap/engine.hpp:58-59
 *   TvolapEngine::exchange_filter(next)             proj/include/tvolap/engine.hpp:55-56
 *   TvolapEngine::reset / op_counts / getters       proj/include/tvolap/engine.hpp:38-50,62-64
 *   TvolapProcessor(ir, hop) / set_filter(ir)       proj/include/tvolap/reference.hpp:202-221
 *   forward_real / inverse_real / mac               proj/include/tvolap/spectral.hpp:36-47
 *   hann_window                                     proj/include/tvolap/partition.hpp:16
 *
 * Plain pointers and sizes only. Sample data is fp32, planar, one lane after
 * another: sample t of lane c lives at ptr[c * lane_stride + t] (the
 * column-per-channel layout of proj/include/tvolap/audio_buffer.hpp:11-15).
 * Every pointer argument may be host memory (pageable or pinned) or device
 * memory of the engine's GPU; the engine detects which. Calls on device
 * pointers are asynchronous on the engine's stream (see tvolap_set_stream /
 * tvolap_synchronize); calls on host pointers return when the host output is
 * written, like the reference's by-value return.
 *
 * Every entry point returns a status; the non-zero codes map one-to-one onto
 * the reference's exception classes (proj/include/tvolap/errors.hpp:10-62).
 * tvolap_last_error() gives the message of the calling thread's last failure.
 * There is no CPU fallback: without a usable sm_100 device every call that
 * needs one fails with TVOLAP_ERR_CUDA.
 */
#ifndef TVOLAP_B200_H
#define TVOLAP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TVOLAP_OK 0
#define TVOLAP_ERR_INVALID_SIZE 1          /* tvolap::InvalidSizeError          errors.hpp:10-13 */
#define TVOLAP_ERR_INVALID_INPUT 2         /* tvolap::InvalidInputError         errors.hpp:16-19 */
#define TVOLAP_ERR_INVALID_CONFIGURATION 3 /* tvolap::InvalidConfigurationError errors.hpp:40-43 */
#define TVOLAP_ERR_INCOMPATIBLE_FILTER 4   /* tvolap::IncompatibleFilterError   errors.hpp:34-37 */
#define TVOLAP_ERR_INVALID_SPECTRUM 5      /* tvolap::InvalidSpectrumError      errors.hpp:28-31 */
#define TVOLAP_ERR_CUDA 6                  /* device / driver failure (no reference analogue) */

typedef struct tvolap_engine tvolap_engine;
typedef struct tvolap_set tvolap_set;

/* Message for the calling thread's most recent failing call. */
const char* tvolap_last_error(void);

/* Library version string and the sm_100a build tag. */
const char* tvolap_version(void);

/* ---------------------------------------------------------------- engines */

/*
 * Filter-set engine: TvolapProcessor(ir, hop) ≙ TvolapEngine(partition(ir, hop,
 * min_partitions)) (reference.cpp:328-329, partition.cpp:20-51, engine.cpp:9-32).
 * ir: channels impulse responses of ir_length taps, ir[c * ir_length + n].
 * M = max(ceil(ir_length / 2L), min_partitions). Errors: INVALID_INPUT for an
 * empty IR (partition.cpp:21-22), INVALID_SIZE when 4L is not a power of two
 * or L < 2 (partition.cpp:23-24).
 */
int tvolap_create(tvolap_engine** out, int device, long hop, long channels, long ir_length, const float* ir,
                  long min_partitions);

/*
 * Bank engine (BASELINE configs C1/C3/C5): `sources` input streams, each fanned
 * out to `ears` lanes (audio_buffer.hpp:60-67 fan_out, fused so the ears share
 * one input spectrum). The filter pool is a pre-partitioned bank of n_bank
 * entries, bank_ir[(b * ears + e) * ir_length + n]; every source selects one
 * entry per hop (the zero-copy exchange_filter(shared_ptr) of engine.hpp:55
 * with pre-built sets). All sources start on entry 0.
 */
int tvolap_create_bank(tvolap_engine** out, int device, long hop, long sources, long ears, long n_bank,
                       long ir_length, const float* bank_ir, long min_partitions);

int tvolap_destroy(tvolap_engine* e);

/*
 * One hop: TvolapEngine::process (engine.cpp:60-106). in: L samples for each of
 * `channels` (= sources) lanes; out: L samples for each of channels*ears output
 * lanes (lane s*ears + e). A staged filter / bank selection is latched first
 * (engine.cpp:61). rows must equal L (INVALID_SIZE, engine.cpp:64-65) and cols
 * the input channel count (INVALID_INPUT, engine.cpp:66-67).
 */
int tvolap_process(tvolap_engine* e, const float* in, long in_lane_stride, long rows, long cols, float* out,
                   long out_lane_stride);

/*
 * n_hops consecutive hops — semantically n_hops process() calls (the
 * reference's drive() loop, experiment.cpp:43-49). in/out hold n_hops*L
 * samples per lane. schedule (bank engines only, may be NULL) gives the bank
 * entry of every (hop, source): schedule[h * sources + s]; when NULL the
 * current selection holds for all hops. Host pointers are streamed through
 * pinned staging buffers with copies overlapping the kernels. With few channels
 * (channels x cluster CTAs <= 2 per SM) the hops run as time-parallel passes
 * (filter-set engines: calls of >= 32 hops; bank engines: schedules that only
 * change every >= 3 hops), bit-identical to the hop-blocked launch and to
 * process(); tvolap_wide_passes counts them.
 */
int tvolap_process_hops(tvolap_engine* e, const float* in, long in_lane_stride, float* out, long out_lane_stride,
                        long n_hops, const int32_t* schedule);

/*
 * n_hops hops with a filter switch every `period` hops: exactly
 *   for k: { if (irs[k]) exchange_filter(irs[k], ir_length, channels); process_hops(period) }
 * (the reference's drive() loop, experiment.cpp:42-49, with the switch staged right before the
 * hop it applies to), k < ceil(n_hops / period); irs[k] == NULL keeps the running filter. `irs`
 * is a host array of channel-major IR pointers (irs[k][c * ir_length + n]). With device
 * buffers and device IRs the call runs as a time-parallel pass when the engine has few channels
 * (forward FFTs of every hop at once, then one CTA per (channel, period) that transforms its
 * period's set in-CTA and runs MAC + inverse + overlap-add; tvolap_wide_passes counts them), or
 * as one hop-blocked launch that transforms switch k+1's partitions inside the cluster-barrier
 * gaps of period k; otherwise it runs the loop above. The hop-blocked forms are bit-identical to
 * the loop; the time-parallel pass is too with TVOLAP_WIDE_WARPFFT=0, and by default (warp
 * per-frame transforms) equal to fp32 rounding. Filter-set engines only.
 */
int tvolap_process_switching(tvolap_engine* e, const float* in, long in_lane_stride, float* out, long out_lane_stride,
                             long n_hops, long period, const float* const* irs, long ir_length);

/*
 * Stage a replacement filter: TvolapProcessor::set_filter(ir) ≙
 * exchange_filter(partition(ir, L, M)) (reference.cpp:335-338,
 * engine.cpp:37-48). The partition runs on the device on a side stream
 * overlapping the running hops; the set is latched at the next process call
 * (last staged wins). Errors: INCOMPATIBLE_FILTER when channels differ or the
 * IR needs more than M partitions (engine.cpp:38-45); INVALID_INPUT for an
 * empty IR. Filter-set engines only (INVALID_CONFIGURATION on a bank engine).
 */
int tvolap_exchange_filter(tvolap_engine* e, const float* ir, long ir_length, long channels);

/*
 * Device-resident filter partition sets: the reference's immutable, shared
 * FilterPartitionSet (partition.hpp:21-32) held on the GPU.
 *   tvolap_set_create   ≙ partition(ir, hop, min_partitions) (partition.hpp:38, partition.cpp:20-51):
 *                         K4 once, on `device`; errors as tvolap_create. Reference-counted: the
 *                         caller owns one reference (tvolap_set_release); an engine holding the set
 *                         as its active or staged filter holds another.
 *   tvolap_create_from_set ≙ TvolapEngine(shared_ptr<const FilterPartitionSet>) (engine.hpp:35):
 *                         no transform, the engine reads the set's spectra in place.
 *   tvolap_exchange_set ≙ exchange_filter(shared_ptr<const FilterPartitionSet>) (engine.hpp:55,
 *                         engine.cpp:37-48): O(1), no K4; validated (INCOMPATIBLE_FILTER on a hop,
 *                         partition-count, channel-count or device mismatch), latched at the next
 *                         process call, last staged wins (also against tvolap_exchange_filter).
 *   tvolap_set_reassemble ≙ reassemble(set) (partition.hpp:43, partition.cpp:53-65):
 *                         out[c * (2 L M) + n], the response zero-padded to M * 2L taps.
 *   tvolap_set_spectra:   spectra[((c * M + m) * (2L + 1) + k) * 2 + {re, im}] (as tvolap_partition).
 */
int tvolap_set_create(tvolap_set** out, int device, long hop, long channels, long ir_length, const float* ir,
                      long min_partitions);
int tvolap_set_release(tvolap_set* s);
int tvolap_set_geometry(const tvolap_set* s, long* hop, long* partitions, long* channels, long* source_length);
int tvolap_set_spectra(const tvolap_set* s, float* spectra);
int tvolap_set_reassemble(const tvolap_set* s, float* out);
int tvolap_create_from_set(tvolap_engine** out, const tvolap_set* s);
int tvolap_exchange_set(tvolap_engine* e, const tvolap_set* s);

/* Stage per-source bank selections idx[sources], latched at the next hop. */
int tvolap_select_bank(tvolap_engine* e, const int32_t* idx);

/* TvolapEngine::reset (engine.cpp:108-118): zero all state, keep any staged filter. */
int tvolap_reset(tvolap_engine* e);

/* Getters: engine.hpp:38-50. */
long tvolap_hop(const tvolap_engine* e);
long tvolap_channels(const tvolap_engine* e);        /* input channels (sources) */
long tvolap_output_channels(const tvolap_engine* e); /* channels * ears */
long tvolap_partition_count(const tvolap_engine* e);
long tvolap_delay_line_depth(const tvolap_engine* e); /* 2M-1 */
long tvolap_latency(const tvolap_engine* e);          /* 2L */
long tvolap_switching_latency(const tvolap_engine* e);/* L */
long tvolap_stream_delay(const tvolap_engine* e);     /* L */
long tvolap_hops_processed(const tvolap_engine* e);

/*
 * EngineOpCounts (engine.hpp:17-21): cumulative forward transforms, inverse
 * transforms and spectral MACs actually executed. For ears == 1 these equal the
 * reference's per-channel counts; with ears == 2 one forward transform serves
 * both ears of a source.
 */
int tvolap_op_counts(const tvolap_engine* e, uint64_t* forward, uint64_t* inverse, uint64_t* macs);

/* Engine stream control. `stream` is a cudaStream_t passed as void*; NULL restores the engine's own. */
int tvolap_set_stream(tvolap_engine* e, void* stream);
int tvolap_synchronize(tvolap_engine* e);

/*
 * Throughput mode for pinned host buffers: when enabled, process / process_hops
 * on pinned (cudaHostAlloc / cudaHostRegister) host memory return once the
 * copies and kernels are queued, like cudaMemcpyAsync; tvolap_synchronize()
 * waits for the outputs. exchange_filter from pinned memory is always
 * asynchronous (the buffer must stay untouched until the next process call
 * has been synchronized). Pageable host memory is always synchronous.
 */
int tvolap_set_host_async(tvolap_engine* e, int enable);

/*
 * Kernel timing: while enabled, every fused hop-kernel launch is bracketed by
 * CUDA events on the launching stream. tvolap_kernel_time() waits for them and
 * returns the summed device time and the number of launches since profiling
 * was enabled (or last read), then starts a new window.
 */
int tvolap_set_profiling(tvolap_engine* e, int enable);
int tvolap_kernel_time(tvolap_engine* e, double* total_ms, long* launches);

/* Launch configuration: CTAs per source (thread-block cluster size) of the multi-hop (blocked)
 * kernel and threads per CTA the one-hop kernel is launched with (the automatic rule, or the
 * override below / tuning "nt"; every value gives the same output bits). */
int tvolap_launch_config(const tvolap_engine* e, int* ctas_per_source, int* threads_per_cta);
/* Override the cluster size P (1, 2, 4 or 8; both kernels) and the one-hop kernel's threads per CTA
 * (32..1024); 0 keeps the current value. */
int tvolap_set_launch_config(tvolap_engine* e, int ctas_per_source, int threads_per_cta);

/*
 * Hop blocking for multi-hop calls: process_hops calls with at least block_min
 * hops run the hop-blocked kernel, which processes hops_per_block (2, 4, 8, 16)
 * consecutive hops together and loads each delay-line / shared filter slice
 * once per block instead of once per hop. Outputs are the same per-hop sums;
 * 0 keeps the current value.
 */
int tvolap_set_block_config(tvolap_engine* e, int hops_per_block, long block_min);
int tvolap_block_config(const tvolap_engine* e, int* hops_per_block, long* block_min, int* partition_groups);

/* Number of kernels this engine has launched since creation. */
uint64_t tvolap_kernel_launches(const tvolap_engine* e);

/* Time-parallel passes run so far: device-resident tvolap_process_switching calls executed as
   K1-for-all-hops + (lane, hop-tile) K4/MAC/inverse CTAs, and bank passes of per-hop bank
   schedules (a diagnostic of which path a call took; tuning "wide" / "bank_pass" select). */
uint64_t tvolap_wide_passes(const tvolap_engine* e);

/* One-hop launches of bank engines that ran on the persistent bulk-copy ring kernel (delay-line
   and filter rows staged into shared memory by cp.async.bulk + mbarrier across sources; tuning
   "hop_ring"); the others ran on the cluster hop kernel. A diagnostic like tvolap_wide_passes. */
uint64_t tvolap_ring_launches(const tvolap_engine* e);

/*
 * Tuning knobs: every A/B switch of the kernel, geometry and pipeline choices, by name (the
 * library reads no environment variables). Defaults are the measured-best choices; DESIGN.md §10
 * documents each key. Engine knobs apply to that engine; "pdl", "k4_warp" and "k4_prefetch" are
 * process-wide launch knobs. Unknown keys and out-of-range values return INVALID_INPUT; a
 * geometry that does not fit returns INVALID_CONFIGURATION and keeps the previous value.
 * tvolap_set_default_tuning sets the value engines created afterwards start with.
 * No reference counterpart (the reference has no tunables).
 */
int tvolap_set_tuning(tvolap_engine* e, const char* key, long value);
int tvolap_get_tuning(const tvolap_engine* e, const char* key, long* value);
int tvolap_set_default_tuning(const char* key, long value);
int tvolap_reset_default_tuning(void);
/* Comma-separated list of the keys. */
const char* tvolap_tuning_keys(void);

/* ------------------------------------------------------ spectral primitives */
/* Batched K1/K5 building blocks, exposed so the reference's spectral tests
 * (proj/tests/test_spectral.cpp) run against the device FFT. */

/* forward_real (spectral.cpp:99-125): x[b * n + i] -> bins[(b * (n/2+1) + k) * 2 + {re,im}].
 * n must be a power of two >= 8 (INVALID_SIZE otherwise). */
int tvolap_forward_real(int device, long n, long batch, const float* x, float* bins);

/* inverse_real (spectral.cpp:127-158): bins -> x, with the 1/n scaling.
 * INVALID_SPECTRUM if a DC or Nyquist bin has a non-zero imaginary part. */
int tvolap_inverse_real(int device, long n, long batch, const float* bins, float* x);

/* mac (spectral.cpp:160-172): out = acc + a*b over nbins complex bins, batch frames. */
int tvolap_mac(int device, long nbins, long batch, const float* acc, const float* a, const float* b, float* out);

/* hann_window (partition.cpp:10-18), computed in fp64 and rounded: w[2L]. */
int tvolap_hann_window(long hop, float* w);

/*
 * partition (partition.cpp:20-51) on the device: spectra[((c * M + m) * (2L+1) + k) * 2 + {re,im}],
 * M = max(ceil(ir_length / 2L), min_partitions) returned in *partitions.
 */
int tvolap_partition(int device, long hop, long channels, long ir_length, const float* ir, long min_partitions,
                     float* spectra, long* partitions);

/* ------------------------------------------------------ device workload helpers */
/* Fill device memory with the seeded generators of workload.h (the same values the
 * host twin libtvolap_workload.so produces). Used by the benchmark to keep
 * inputs resident in HBM; not part of the reference boundary. */
int tvolap_gen_white_device(int device, uint64_t seed, long lane0, long lanes, long t0, long n, float* out,
                            long stride);
int tvolap_gen_irs_device(int device, uint64_t seed, long count, const long* lanes, const long* ears,
                          const long* ks, const double* t60, double fs, long len, float* out);

/* Binaural mix (config C3): mix[e * mix_stride + t] = sum_s out[(s * ears + e) * out_stride + t],
 * summed in a fixed order (deterministic). Device pointers. */
int tvolap_mix_device(int device, long sources, long ears, long samples, const float* out, long out_stride,
                      float* mix, long mix_stride, void* stream);

/*
 * Multi-GPU C3 mix (sources sharded across GPUs, the stereo mix reduced with NCCL
 * over NVLink): this GPU's partial mix of its own sources (tvolap_mix_device) followed by an
 * in-place ncclAllReduce(sum) of the ears x samples partial mix over `nccl_comm`, both on `stream`.
 * nccl_comm == NULL: the single-GPU mix only. `nccl_comm` is an ncclComm_t (void* so this header
 * does not need nccl.h); NCCL is loaded at first use (libnccl.so.2), so hosts that never mix
 * carry no NCCL dependency. No reference counterpart (the reference mixes on one CPU thread).
 */
int tvolap_mix_allreduce(int device, long sources, long ears, long samples, const float* out, long out_stride,
                         float* mix, long mix_stride, void* nccl_comm, void* stream);
/* Communicator helpers for hosts without their own NCCL setup: rank 0 makes the 128-byte unique
 * id, the host distributes it (any transport), every rank calls tvolap_nccl_comm_init. */
int tvolap_nccl_unique_id(char id_out[128]);
int tvolap_nccl_comm_init(void** comm_out, int device, int nranks, int rank, const char id[128]);
int tvolap_nccl_comm_destroy(void* comm);


/*
 * Multi-GPU C3 mix over peer memory (the fused alternative to tvolap_mix_allreduce): one kernel per
 * rank sums the GPU's sources and stores the partial mix straight into slot `rank` of every rank's
 * gather buffer (NVLink P2P stores into cudaIpc-mapped peer buffers); a second kernel sums the
 * slots in rank order, so every rank ends with the bit-identical mix. Setup: every rank creates its
 * group (its gather buffer + a 64-byte IPC handle), the host distributes the handles (any
 * transport), every rank opens them. Per pass: tvolap_mix_scatter on every rank; all ranks'
 * scatters complete (stream sync + a host barrier); tvolap_mix_gather; a host barrier before the
 * next scatter overwrites the slots. world == 1 needs no handles. Replaces the per-GPU sum +
 * ncclAllReduce of the reference's single-process mix (audio_buffer.hpp:60-67 summed per GPU).
 */
typedef struct tvolap_mix_group tvolap_mix_group;
int tvolap_mix_group_create(tvolap_mix_group** out, int device, int world, int rank, long ears, long capacity,
                            char ipc_handle_out[64]);
int tvolap_mix_group_open(tvolap_mix_group* g, const char* handles /* world x 64 bytes, rank order */);
int tvolap_mix_scatter(tvolap_mix_group* g, long sources, long samples, const float* out, long out_stride,
                       void* stream);
int tvolap_mix_gather(tvolap_mix_group* g, long samples, float* mix, long mix_stride, void* stream);
int tvolap_mix_group_destroy(tvolap_mix_group* g);

/* ------------------------------------------------------ comparison convolvers
 * The reference's other streaming convolvers (reference.hpp:53-200, reference.cpp:34-320) on the
 * GPU, for switching comparisons against TVOLAP:
 *   TVOLAP_CMP_TDC    DirectProcessor "tdc"    direct-form FIR, hard switch at hop boundaries
 *   TVOLAP_CMP_CF_TDC CfTdcProcessor "cf-tdc"  direct form with a crossfade of the two outputs
 *   TVOLAP_CMP_OLA    OlaProcessor "ola"       block = IR length, hop = block
 *   TVOLAP_CMP_OLS    OlsProcessor "ols"       block = IR length, hop = block
 *   TVOLAP_CMP_WOLA   WolaProcessor "wola"     sqrt-Hann analysis/synthesis, hop = block / 2
 * ir is channel-major (ir[c * ir_stride + t], t < taps). "tdc"/"cf-tdc" take `hop`; the block
 * forms need a power-of-two taps >= 4 (GPU limit: taps <= 4096). Errors as the reference's
 * constructors / set_filter / switch_filter (InvalidSize, InvalidInput, InvalidConfiguration,
 * IncompatibleFilter, SwitchInProgress). Calls are synchronous; buffers may be host or device. */
#define TVOLAP_ERR_SWITCH_IN_PROGRESS 7    /* tvolap::SwitchInProgressError     errors.hpp:46-49 */
#define TVOLAP_CMP_TDC 0
#define TVOLAP_CMP_CF_TDC 1
#define TVOLAP_CMP_OLA 2
#define TVOLAP_CMP_OLS 3
#define TVOLAP_CMP_WOLA 4
#define TVOLAP_FADE_HANN 0   /* CrossfadeConfig::Shape::HannComplementary (reference.hpp:19) */
#define TVOLAP_FADE_LINEAR 1 /* CrossfadeConfig::Shape::Linear */
typedef struct tvolap_cmp tvolap_cmp;

/* Constructors (reference.cpp:59-66, 97-108, 184-190, 221-227, 259-267). */
int tvolap_cmp_create(tvolap_cmp** out, int device, int kind, long taps, long channels, const float* ir,
                      long ir_stride, long hop, long fade_duration, int fade_shape);
int tvolap_cmp_destroy(tvolap_cmp* p);
/* n_hops consecutive process() calls (reference.cpp:68-93, 136-172, 192-216, 229-252, 269-308):
 * in[c * in_stride + t], out[c * out_stride + t], t < n_hops * hop. */
int tvolap_cmp_process_hops(tvolap_cmp* p, const float* in, long in_stride, float* out, long out_stride,
                            long n_hops);
/* set_filter (reference.cpp:78-82, 134-136, 192-196, 229-233, 269-273): staged, applied at the next hop. */
int tvolap_cmp_set_filter(tvolap_cmp* p, const float* ir, long taps, long channels, long ir_stride);
/* CfTdcProcessor::switch_filter (reference.cpp:122-132). */
int tvolap_cmp_switch_filter(tvolap_cmp* p, const float* ir, long taps, long channels, long ir_stride,
                             long fade_duration, int fade_shape);
int tvolap_cmp_reset(tvolap_cmp* p);
/* out6 = {hop, channels, latency, stream_delay, switching_latency, fading} (reference.hpp:53-200). */
int tvolap_cmp_geometry(const tvolap_cmp* p, long* out6);

#ifdef __cplusplus
}
#endif

#endif /* TVOLAP_B200_H */
