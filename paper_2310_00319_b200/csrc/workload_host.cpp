// Host twin of the seeded workload generators (workload.h). Builds into
// libtvolap_workload.so (plain C++, no CUDA) so CPU tests, the oracle legs of
// bench.py and the e2e host buffers all see the exact inputs the device
// generators produce. Not part of the hot path.
#include <algorithm>
#include <cmath>
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

}  // extern "C"
