// Seeded synthetic workload generators shared bit-for-bit by the host (C++,
// feeding the oracle and pinned host buffers) and the device (CUDA kernels
// that fill HBM directly). Integer-exact counter-based RNG, so any (seed,
// stream, counter) triple yields the same 64-bit word on both sides.
//
// The uniform mapping is the reference's 53-bit one,
// 2 * ((g() >> 11) * 2^-53) - 1  (proj/src/signal_gen.cpp:14-16); only the
// 64-bit source differs (a SplitMix64-style counter hash instead of a
// sequential mt19937_64), because a counter generator can be evaluated in
// parallel on the GPU. Gaussians are Box-Muller on two such words (portable,
// unlike std::normal_distribution — SURVEY.md §7 step 1). Decay envelopes
// follow BASELINE.json: Gaussian * exp(-6.91 n / (T60 fs)), unit energy.
#pragma once

#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define TV_HD __host__ __device__ __forceinline__
#else
#define TV_HD static inline
#endif

TV_HD uint64_t tv_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// One 64-bit word for (seed, stream, counter).
TV_HD uint64_t tv_rand64(uint64_t seed, uint64_t stream, uint64_t ctr) {
    const uint64_t key = tv_mix64(seed * 0x9E3779B97F4A7C15ULL + tv_mix64(stream + 0x632BE59BD9B4E019ULL));
    return tv_mix64(key + (ctr + 1) * 0x9E3779B97F4A7C15ULL);
}

// signal_gen.cpp:14-16 mapping: uniform in [-1, 1).
TV_HD double tv_uniform_pm1(uint64_t r) { return 2.0 * ((double)(r >> 11) * 0x1.0p-53) - 1.0; }

// Uniform in [0, 1).
TV_HD double tv_uniform01(uint64_t r) { return (double)(r >> 11) * 0x1.0p-53; }

// Box-Muller standard normal from counters 2n and 2n+1 of (seed, stream).
TV_HD double tv_gauss(uint64_t seed, uint64_t stream, uint64_t n) {
    const double u1 = ((double)(tv_rand64(seed, stream, 2 * n) >> 11) + 1.0) * 0x1.0p-53;  // (0, 1]
    const double u2 = tv_uniform01(tv_rand64(seed, stream, 2 * n + 1));
    return sqrt(-2.0 * log(u1)) * cos(6.283185307179586476925286766559 * u2);
}

// Stream ids: white-noise input of lane `lane`; IR `k` of (lane, ear).
TV_HD uint64_t tv_stream_input(uint64_t lane) { return (1ULL << 60) | lane; }
TV_HD uint64_t tv_stream_ir(uint64_t lane, uint64_t ear, uint64_t k) {
    return (2ULL << 60) | (lane << 28) | (ear << 24) | k;
}
TV_HD uint64_t tv_stream_t60(uint64_t lane, uint64_t k) { return (3ULL << 60) | (lane << 24) | k; }
TV_HD uint64_t tv_stream_sched(uint64_t hop) { return (4ULL << 60) | hop; }

// Unnormalised decaying-noise tap n of an IR with reverberation time t60.
TV_HD double tv_ir_tap(uint64_t seed, uint64_t stream, uint64_t n, double t60, double fs) {
    return tv_gauss(seed, stream, n) * exp(-6.91 * (double)n / (t60 * fs));
}

// T60 drawn uniformly from [lo, hi] for (lane, k).
TV_HD double tv_t60(uint64_t seed, uint64_t lane, uint64_t k, double lo, double hi) {
    return lo + (hi - lo) * tv_uniform01(tv_rand64(seed, tv_stream_t60(lane, k), 0));
}

// Bank choice of `lane` at `hop`, uniform over n_bank entries.
TV_HD int tv_choice(uint64_t seed, uint64_t hop, uint64_t lane, int n_bank) {
    return (int)(tv_uniform01(tv_rand64(seed, tv_stream_sched(hop), lane)) * (double)n_bank);
}
