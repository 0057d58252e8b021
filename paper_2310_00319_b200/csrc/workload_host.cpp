// Host twin of the seeded workload generators (workload.h). Builds into
// libtvolap_workload.so (plain C++, no CUDA) so CPU tests, the oracle legs of
// bench.py and the e2e host buffers all see the exact inputs the device
// generators produce. Not part of the hot path.
#include <algorithm>
#include <cmath>
#include <random>
#include <cstdint>
#include <thread>
#include <vector>

#include "workload.h"

namespace {

template <class F>
void parallel_for(long n, int threads, F&& f) {
    if (threads <= 1 || n <= 1) {
        for (long i = 0; i < n; ++i) f(i);
        return;
    }
    std::vector<std::thread> pool;
    const long per = (n + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const long a = t * per, b = std::min(n, a + per);
        if (a < b)
            pool.emplace_back([&, a, b] {
                for (long i = a; i < b; ++i) f(i);
            });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

// White noise, uniform [-1, 1): out[l * stride + t] for lanes lane0..lane0+lanes-1,
// samples t0..t0+n-1 of each lane's stream. Either output may be null.
void tv_gen_white(uint64_t seed, long lane0, long lanes, long t0, long n, float* out32, double* out64, long stride,
                  int threads) {
    parallel_for(lanes, threads, [&](long l) {
        const uint64_t st = tv_stream_input((uint64_t)(lane0 + l));
        for (long t = 0; t < n; ++t) {
            const double v = tv_uniform_pm1(tv_rand64(seed, st, (uint64_t)(t0 + t)));
            if (out32) out32[l * stride + t] = (float)v;
            if (out64) out64[l * stride + t] = (double)(float)v;
        }
    });
}

// Unit-energy decaying-noise IRs for a list of (lane, ear, k) triples with per-item
// T60; item i writes out[i * len ...]. out64 receives the fp32-rounded values so
// both the oracle and the GPU see identical taps.
void tv_gen_irs(uint64_t seed, long count, const long* lanes, const long* ears, const long* ks, const double* t60,
                double fs, long len, float* out32, double* out64, int threads) {
    parallel_for(count, threads, [&](long i) {
        const uint64_t st = tv_stream_ir((uint64_t)lanes[i], (uint64_t)ears[i], (uint64_t)ks[i]);
        std::vector<double> h(len);
        double e = 0.0;
        for (long n = 0; n < len; ++n) {
            h[n] = tv_ir_tap(seed, st, (uint64_t)n, t60[i], fs);
            e += h[n] * h[n];
        }
        const double g = e > 0.0 ? 1.0 / std::sqrt(e) : 0.0;
        for (long n = 0; n < len; ++n) {
            const float v = (float)(h[n] * g);
            if (out32) out32[i * len + n] = v;
            if (out64) out64[i * len + n] = (double)v;
        }
    });
}

double tv_t60_c(uint64_t seed, long lane, long k, double lo, double hi) {
    return tv_t60(seed, (uint64_t)lane, (uint64_t)k, lo, hi);
}

// Per-hop bank choices: out[h * lanes + l] for hops hop0..hop0+n_hops-1.
void tv_gen_schedule(uint64_t seed, long hop0, long n_hops, long lanes, int n_bank, int* out, int threads) {
    parallel_for(n_hops, threads, [&](long h) {
        for (long l = 0; l < lanes; ++l)
            out[h * lanes + l] = tv_choice(seed, (uint64_t)(hop0 + h), (uint64_t)l, n_bank);
    });
}

uint64_t tv_rand64_c(uint64_t seed, uint64_t stream, uint64_t ctr) { return tv_rand64(seed, stream, ctr); }


// ---- the reference's CLI signal generators (proj/src/signal_gen.cpp), with the same engine
// (std::mt19937_64) and the same 53-bit mapping (signal_gen.cpp:14-16), so `pink:SEED` and
// `synth:azDEG` specs produce the reference's exact fp64 streams.
static double tv_uniform_pm1(std::mt19937_64& g) { return 2.0 * ((double)(g() >> 11) * 0x1.0p-53) - 1.0; }

// gen_pink (signal_gen.cpp:42-59): Kellet's pole-zero cascade over uniform white noise.
void tv_gen_pink(uint64_t seed, long n, double* out) {
    std::mt19937_64 g(seed);
    double b0 = 0, b1 = 0, b2 = 0, b3 = 0, b4 = 0, b5 = 0, b6 = 0;
    for (long t = 0; t < n; ++t) {
        const double w = tv_uniform_pm1(g);
        b0 = 0.99886 * b0 + w * 0.0555179;
        b1 = 0.99332 * b1 + w * 0.0750759;
        b2 = 0.96900 * b2 + w * 0.1538520;
        b3 = 0.86650 * b3 + w * 0.3104856;
        b4 = 0.55000 * b4 + w * 0.5329522;
        b5 = -0.7616 * b5 - w * 0.0168980;
        out[t] = 0.11 * (b0 + b1 + b2 + b3 + b4 + b5 + b6 + w * 0.5362);
        b6 = w * 0.115926;
    }
}

// synthetic_binaural_ir (signal_gen.cpp:73-107): direct taps with an azimuth-dependent
// interaural delay / level, plus a shared decaying room tail 30 dB down. out[c * n_ir + q].
int tv_synthetic_binaural_ir(double azimuth_deg, long n_ir, double fs, uint64_t seed, double* out) {
    if (n_ir < 128 || !(fs > 0.0)) return 2;
    const double pi = 3.14159265358979323846264338327950288;
    for (long i = 0; i < 2 * n_ir; ++i) out[i] = 0.0;
    const double lateral = std::sin(azimuth_deg * pi / 180.0);
    const long base_delay = 2;
    const long max_itd = (long)std::llround(fs / 1500.0);
    const long itd = (long)std::llround(std::fabs(lateral) * (double)max_itd);
    const double far_gain = itd == 0 ? 1.0 : 1.0 - 0.75 * std::fabs(lateral);
    const long near = lateral >= 0.0 ? 0 : 1;
    out[near * n_ir + base_delay] = 1.0;
    out[(1 - near) * n_ir + base_delay + itd] = far_gain;
    const long tail_start = 64;
    const double tau = (double)std::max<long>(256, n_ir / 8);
    for (long c = 0; c < 2; ++c) {
        std::mt19937_64 g(seed ^ (0x9e3779b97f4a7c15ULL * (uint64_t)(c + 1)));
        for (long q = tail_start; q < n_ir; ++q)
            out[c * n_ir + q] += 0.0316 * std::exp(-(double)(q - tail_start) / tau) * tv_uniform_pm1(g);
    }
    return 0;
}

}  // extern "C"
