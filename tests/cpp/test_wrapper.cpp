// Drop-in check of include/tvolap_b200.hpp: the reference's own engine tests
// (proj/tests/test_engine.cpp:71-77 identity, :159-188 half-cosine crossfade,
// :203-216 error classes, partition/reassemble of test_partition.cpp) written
// against the C++ wrapper exactly as the reference writes them against
// tvolap::TvolapEngine; run by tests/test_gpu_engine.py::test_cpp_wrapper. Exit 0 = pass,
// 77 = no GPU (the wrapper threw CudaError: there is no CPU fallback).
#include <cmath>
#include <cstdio>
#include <memory>

#include "tvolap_b200.hpp"

using namespace tvolap_b200;

static ImpulseResponse delta_ir(double gain, Index len) {
    ImpulseResponse ir;
    ir.samples = Frames(len, 1);
    ir.samples(0, 0) = gain;
    return ir;
}

static int fails = 0;
#define CHECK(c)                                                   \
    do {                                                           \
        if (!(c)) {                                                \
            std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); \
            ++fails;                                               \
        }                                                          \
    } while (0)

int main() {
    try {
        // identity passthrough, L = 16
        TvolapEngine id(partition(delta_ir(1.0, 1), 16));
        Frames x(16, 1);
        double worst = 0.0;
        for (int h = 0; h < 10; ++h) {
            for (Index i = 0; i < 16; ++i) x(i, 0) = std::sin(0.37 * (h * 16 + i));
            Frames y = id.process(x);
            if (h > 0)
                for (Index i = 0; i < 16; ++i) worst = std::fmax(worst, std::fabs(y(i, 0) - std::sin(0.37 * (h * 16 + i - 16))));
        }
        CHECK(worst < 1e-5);

        // polarity flip crosses over along the half-cosine
        const Index hop = 256;
        TvolapEngine eng(partition(delta_ir(1.0, 2048), hop));
        CHECK(eng.partition_count() == 4 && eng.delay_line_depth() == 7 && eng.latency() == 512);
        Frames ones(hop, 1, 1.0);
        std::vector<double> stream;
        for (int i = 0; i < 24; ++i) {
            if (i == 12) eng.exchange_filter(partition(delta_ir(-1.0, 2048), hop));
            Frames y = eng.process(ones);
            for (Index u = 0; u < hop; ++u) stream.push_back(y(u, 0));
        }
        const Index boundary = 11 * hop + hop;  // + stream_delay
        const double pi = 3.14159265358979323846;
        double cerr = 0.0;
        for (Index u = 0; u < hop; ++u) cerr = std::fmax(cerr, std::fabs(stream[boundary + u] - std::cos(pi * u / hop)));
        CHECK(cerr < 1e-5);
        CHECK(std::fabs(stream.back() + 1.0) < 1e-5);
        EngineOpCounts c = eng.op_counts();
        CHECK(c.forward_transforms == 24 && c.inverse_transforms == 24 && c.spectral_macs == 96);

        // error classes
        bool threw = false;
        try { eng.process(Frames(hop - 1, 1)); } catch (const InvalidSizeError&) { threw = true; }
        CHECK(threw);
        threw = false;
        try { eng.process(Frames(hop, 2)); } catch (const InvalidInputError&) { threw = true; }
        CHECK(threw);
        threw = false;
        try { eng.exchange_filter(partition(delta_ir(1.0, 4096), hop)); } catch (const IncompatibleFilterError&) { threw = true; }
        CHECK(threw);
        threw = false;
        try { TvolapEngine bad(std::shared_ptr<const FilterPartitionSet>{}); } catch (const InvalidConfigurationError&) { threw = true; }
        CHECK(threw);

        // pre-partitioned sets (partition.hpp:21-43): exchange is O(1) — no transform is launched, one
        // set is shared by two engines, reassemble() returns the response zero-padded to M * 2L
        {
            const Index L = 64;
            ImpulseResponse r;
            r.samples = Frames(700, 2);
            for (Index n = 0; n < 700; ++n) {
                r.samples(n, 0) = std::sin(0.1 * n) * std::exp(-n / 200.0);
                r.samples(n, 1) = std::cos(0.07 * n) * std::exp(-n / 150.0);
            }
            auto a = std::make_shared<const FilterPartitionSet>(partition(r, L));
            auto b = std::make_shared<const FilterPartitionSet>(partition(delta_ir(1.0, 700), L));  // 1 channel
            auto d = std::make_shared<const FilterPartitionSet>(partition(r, L, 1));
            TvolapEngine e1(a), e2(a);  // shared
            Frames xin(L, 2, 0.5);
            e1.process(xin);
            const uint64_t before = tvolap_kernel_launches(e1.handle());
            e1.exchange_filter(d);
            e1.process(xin);
            CHECK(tvolap_kernel_launches(e1.handle()) - before == 1);  // the hop kernel only, no K4
            bool t2 = false;
            try { e1.exchange_filter(b); } catch (const IncompatibleFilterError&) { t2 = true; }
            CHECK(t2);
            Frames y2 = e2.process(xin);
            CHECK(y2.rows() == L && y2.cols() == 2);
            ImpulseResponse back = reassemble(*a);
            CHECK(back.length() == 2 * L * a->partition_count && back.channels() == 2);
            double re = 0.0;
            for (Index c = 0; c < 2; ++c)
                for (Index n = 0; n < back.length(); ++n)
                    re = std::fmax(re, std::fabs(back.samples(n, c) - (n < 700 ? r.samples(n, c) : 0.0)));
            CHECK(re < 1e-5);
        }

        TvolapProcessor proc(delta_ir(0.5, 300), 64);
        Frames y = proc.process(Frames(64, 1, 1.0));
        CHECK(proc.name() == "tvolap" && y.rows() == 64);
        proc.set_filter(delta_ir(2.0, 300));  // reference.cpp:335-338: staged, latched next hop
        proc.process(Frames(64, 1, 1.0));
        Frames y3 = proc.process(Frames(64, 1, 1.0));
        CHECK(std::fabs(y3(63, 0) - 2.0) < 1e-5);

        // comparison convolvers through the StreamingProcessor face (reference.hpp:26-226)
        for (const char* name : {"tdc", "cf-tdc", "ola", "ols", "wola", "tvolap"}) {
            auto p = make_processor(name, delta_ir(1.0, 128), 32);
            CHECK(p->name() == name);
            // identity response: after the stream delay the output reproduces the input
            const Index h = p->hop(), d = p->stream_delay();
            std::vector<double> xs, ys;
            for (Index k = 0; k < 8; ++k) {
                Frames x(h, 1);
                for (Index t = 0; t < h; ++t) x(t, 0) = std::sin(0.01 * (double)(k * h + t));
                Frames o = p->process(x);
                for (Index t = 0; t < h; ++t) {
                    xs.push_back(x(t, 0));
                    ys.push_back(o(t, 0));
                }
            }
            double e = 0.0;
            for (size_t t = (size_t)d; t < ys.size(); ++t) e = std::max(e, std::fabs(ys[t] - xs[t - (size_t)d]));
            CHECK(e < 1e-5);
        }
        threw = false;
        try {
            CfTdcProcessor cf(delta_ir(1.0, 8), 32, CrossfadeConfig{200});
            cf.process(Frames(32, 1, 1.0));
            cf.set_filter(delta_ir(0.5, 8));
            cf.set_filter(delta_ir(0.25, 8));
        } catch (const SwitchInProgressError&) { threw = true; }
        CHECK(threw);
    } catch (const CudaError& e) {
        std::printf("NO_GPU %s\n", e.what());
        return 77;
    }
    std::printf(fails ? "FAILED %d\n" : "PASS\n", fails);
    return fails ? 1 : 0;
}
