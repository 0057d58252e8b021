// tvolap_b200.hpp — header-only C++ drop-in over the C-ABI (tvolap_b200.h).
//
// Mirrors the reference's public C++ surface for the hot path so existing
// callers (drive() in proj/src/experiment.cpp:33-54, FrameAdapter in
// proj/src/frame_adapter.cpp:13-43, the CLI's run_process) keep their shape:
//   partition(ir, hop, min_partitions)          proj/include/tvolap/partition.hpp:38
//   FilterPartitionSet                           proj/include/tvolap/partition.hpp:21-32
//   TvolapEngine                                 proj/include/tvolap/engine.hpp:33-94
//   TvolapProcessor / StreamingProcessor face    proj/include/tvolap/reference.hpp:202-221
//   DirectProcessor, CfTdcProcessor, OlaProcessor, OlsProcessor, WolaProcessor,
//   make_processor                               proj/include/tvolap/reference.hpp:26-200,224-226
//   exception classes                            proj/include/tvolap/errors.hpp:10-49
// Eigen is not required: Frames is a minimal column-major (rows = samples,
// cols = channels) fp64 array with the same indexing as Eigen::ArrayXXd, and
// INTEGRATION.md shows the two-line Eigen adapter. Compute is fp32 on the GPU.
#pragma once

#include <algorithm>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "tvolap_b200.h"

namespace tvolap_b200 {

using Index = long;

class InvalidSizeError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class InvalidInputError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class InvalidSpectrumError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class IncompatibleFilterError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class InvalidConfigurationError : public std::invalid_argument {
public:
    using std::invalid_argument::invalid_argument;
};
class CudaError : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};
class SwitchInProgressError : public std::logic_error {
public:
    using std::logic_error::logic_error;
};

inline void check(int rc) {
    if (rc == TVOLAP_OK) return;
    const std::string msg = tvolap_last_error();
    switch (rc) {
        case TVOLAP_ERR_INVALID_SIZE: throw InvalidSizeError(msg);
        case TVOLAP_ERR_INVALID_INPUT: throw InvalidInputError(msg);
        case TVOLAP_ERR_INVALID_CONFIGURATION: throw InvalidConfigurationError(msg);
        case TVOLAP_ERR_INCOMPATIBLE_FILTER: throw IncompatibleFilterError(msg);
        case TVOLAP_ERR_INVALID_SPECTRUM: throw InvalidSpectrumError(msg);
        case TVOLAP_ERR_SWITCH_IN_PROGRESS: throw SwitchInProgressError(msg);
        default: throw CudaError(msg);
    }
}

// Column-major rows x cols array (Eigen::ArrayXXd's storage order).
struct Frames {
    Index rows_ = 0, cols_ = 0;
    std::vector<double> data;
    Frames() = default;
    Frames(Index r, Index c, double fill = 0.0) : rows_(r), cols_(c), data((size_t)(r * c), fill) {}
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    double& operator()(Index r, Index c) { return data[(size_t)(c * rows_ + r)]; }
    double operator()(Index r, Index c) const { return data[(size_t)(c * rows_ + r)]; }
};

struct ImpulseResponse {  // audio_buffer.hpp:30-42
    Frames samples;       // taps x channels
    double sample_rate = 48000.0;
    Index length() const { return samples.rows(); }
    Index channels() const { return samples.cols(); }
};

struct EngineOpCounts {  // engine.hpp:17-21
    std::uint64_t forward_transforms = 0;
    std::uint64_t inverse_transforms = 0;
    std::uint64_t spectral_macs = 0;
};

// partition.hpp:21-32: immutable, shared via shared_ptr. The partition spectra live on the device
// (tvolap_set, computed once by partition()); engines take and exchange to them in O(1). The fp32
// taps it was built from are kept too (TvolapProcessor::set_filter stages taps, whose transform
// then runs on a device side stream).
struct FilterPartitionSet {
    Index hop = 0;
    Index partition_count = 0;
    Index channels = 0;
    Index source_length = 0;
    double normalization_gain = 0.5;
    double sample_rate = 48000.0;
    std::vector<float> taps;             // taps[c * source_length + n]
    std::shared_ptr<tvolap_set> spectra;  // device-resident partition spectra
    int device = 0;
    Index transform_length() const { return 4 * hop; }
    Index padded_length() const { return 2 * hop * partition_count; }
};

inline bool is_power_of_two(Index n) { return n > 0 && (n & (n - 1)) == 0; }

// partition.cpp:20-51: validation and M on the host, the transforms (K4) on the device.
inline FilterPartitionSet partition(const ImpulseResponse& ir, Index hop, Index min_partitions = 1, int device = 0) {
    if (ir.length() < 1 || ir.channels() < 1) throw InvalidInputError("partition: impulse response is empty");
    if (hop < 2 || !is_power_of_two(4 * hop))
        throw InvalidSizeError("partition: 4L must be a power of two, got L = " + std::to_string(hop));
    const Index slice = 2 * hop;
    FilterPartitionSet s;
    s.hop = hop;
    s.partition_count = std::max((ir.length() + slice - 1) / slice, std::max<Index>(min_partitions, 1));
    s.channels = ir.channels();
    s.source_length = ir.length();
    s.sample_rate = ir.sample_rate;
    s.device = device;
    s.taps.resize((size_t)(s.channels * s.source_length));
    for (Index c = 0; c < s.channels; ++c)
        for (Index n = 0; n < s.source_length; ++n) s.taps[(size_t)(c * s.source_length + n)] = (float)ir.samples(n, c);
    tvolap_set* h = nullptr;
    check(tvolap_set_create(&h, device, hop, s.channels, s.source_length, s.taps.data(), s.partition_count));
    s.spectra.reset(h, [](tvolap_set* p) { tvolap_set_release(p); });
    return s;
}

// partition.cpp:53-65: the response zero-padded to M * 2L taps, from the device spectra.
inline ImpulseResponse reassemble(const FilterPartitionSet& set) {
    const Index len = 2 * set.hop * set.partition_count;
    std::vector<float> out((size_t)(len * set.channels));
    check(tvolap_set_reassemble(set.spectra.get(), out.data()));
    ImpulseResponse ir;
    ir.sample_rate = set.sample_rate;
    ir.samples = Frames(len, set.channels);
    for (Index c = 0; c < set.channels; ++c)
        for (Index n = 0; n < len; ++n) ir.samples(n, c) = out[(size_t)(c * len + n)];
    return ir;
}

class TvolapEngine {
public:
    // engine.hpp:35, engine.cpp:9-32: the engine reads the set's device spectra in place
    explicit TvolapEngine(std::shared_ptr<const FilterPartitionSet> filter) : filter_(std::move(filter)) {
        if (!filter_ || !filter_->spectra) throw InvalidConfigurationError("engine requires a filter partition set");
        tvolap_engine* h = nullptr;
        check(tvolap_create_from_set(&h, filter_->spectra.get()));
        h_.reset(h);
    }
    explicit TvolapEngine(const FilterPartitionSet& filter)
        : TvolapEngine(std::make_shared<FilterPartitionSet>(filter)) {}

    Index hop() const { return tvolap_hop(h_.get()); }
    Index channels() const { return tvolap_channels(h_.get()); }
    Index partition_count() const { return tvolap_partition_count(h_.get()); }
    Index delay_line_depth() const { return tvolap_delay_line_depth(h_.get()); }
    Index latency() const { return tvolap_latency(h_.get()); }
    Index switching_latency() const { return tvolap_switching_latency(h_.get()); }
    Index stream_delay() const { return tvolap_stream_delay(h_.get()); }

    // engine.hpp:55, engine.cpp:37-48: O(1) — validate, stage (last wins), latched at the next process()
    void exchange_filter(std::shared_ptr<const FilterPartitionSet> next) {
        if (!next) throw IncompatibleFilterError("replacement filter is null");
        if (next->hop != hop()) throw IncompatibleFilterError("replacement filter hop differs");
        if (next->partition_count != partition_count())
            throw IncompatibleFilterError("replacement filter partition count differs");
        if (next->channels != channels()) throw IncompatibleFilterError("replacement filter channel count differs");
        check(tvolap_exchange_set(h_.get(), next->spectra.get()));
        filter_ = std::move(next);
    }
    void exchange_filter(const FilterPartitionSet& next) { exchange_filter(std::make_shared<FilterPartitionSet>(next)); }
    // TvolapProcessor::set_filter's path: stage time-domain taps; K4 runs on a device side stream
    void exchange_taps(std::shared_ptr<const FilterPartitionSet> next) {
        if (!next) throw IncompatibleFilterError("replacement filter is null");
        check(tvolap_exchange_filter(h_.get(), next->taps.data(), next->source_length, next->channels));
        filter_ = std::move(next);
    }

    // engine.cpp:60-106: exactly L rows x C cols in, same shape out.
    Frames process(const Frames& input) {
        std::vector<float> in((size_t)(input.rows() * input.cols()));
        for (size_t i = 0; i < in.size(); ++i) in[i] = (float)input.data[i];
        std::vector<float> out((size_t)(std::max<Index>(input.rows(), 1) * channels()));
        check(tvolap_process(h_.get(), in.data(), input.rows(), input.rows(), input.cols(), out.data(), input.rows()));
        Frames y(input.rows(), channels());
        for (size_t i = 0; i < y.data.size(); ++i) y.data[i] = out[i];
        return y;
    }

    void reset() { check(tvolap_reset(h_.get())); }

    EngineOpCounts op_counts() const {
        EngineOpCounts c;
        check(tvolap_op_counts(h_.get(), &c.forward_transforms, &c.inverse_transforms, &c.spectral_macs));
        return c;
    }
    const FilterPartitionSet& filter() const { return *filter_; }
    tvolap_engine* handle() const { return h_.get(); }

private:
    struct Del {
        void operator()(tvolap_engine* e) const { tvolap_destroy(e); }
    };
    std::shared_ptr<const FilterPartitionSet> filter_;
    std::unique_ptr<tvolap_engine, Del> h_;
};

// reference.hpp:26-50 — the common face of the streaming convolvers.
class StreamingProcessor {
public:
    virtual ~StreamingProcessor() = default;
    virtual std::string name() const = 0;
    virtual Index hop() const = 0;
    virtual Index channels() const = 0;
    virtual Index latency() const = 0;
    virtual Index stream_delay() const = 0;
    virtual Index switching_latency() const = 0;
    virtual Frames process(const Frames& input) = 0;
    virtual void set_filter(const ImpulseResponse& ir) = 0;
    virtual void reset() = 0;
};

struct CrossfadeConfig {  // reference.hpp:18-22
    enum class Shape { HannComplementary = TVOLAP_FADE_HANN, Linear = TVOLAP_FADE_LINEAR };
    Index duration = 1;
    Shape shape = Shape::HannComplementary;
};

namespace detail {
inline std::vector<float> channel_major(const ImpulseResponse& ir) {
    std::vector<float> t((size_t)(ir.length() * ir.channels()));
    for (Index c = 0; c < ir.channels(); ++c)
        for (Index n = 0; n < ir.length(); ++n) t[(size_t)(c * ir.length() + n)] = (float)ir.samples(n, c);
    return t;
}
struct CmpDel {
    void operator()(tvolap_cmp* p) const { tvolap_cmp_destroy(p); }
};
}  // namespace detail

// The reference's comparison convolvers (reference.hpp:53-200) over tvolap_cmp_* (GPU, fp32).
class CmpProcessor : public StreamingProcessor {
public:
    CmpProcessor(int kind, std::string name, const ImpulseResponse& ir, Index hop, CrossfadeConfig fade, int device)
        : name_(std::move(name)) {
        const std::vector<float> t = detail::channel_major(ir);
        tvolap_cmp* h = nullptr;
        check(tvolap_cmp_create(&h, device, kind, ir.length(), ir.channels(), t.empty() ? nullptr : t.data(),
                                std::max<Index>(ir.length(), 1), hop, fade.duration, (int)fade.shape));
        h_.reset(h);
    }
    std::string name() const override { return name_; }
    Index hop() const override { return geo()[0]; }
    Index channels() const override { return geo()[1]; }
    Index latency() const override { return geo()[2]; }
    Index stream_delay() const override { return geo()[3]; }
    Index switching_latency() const override { return geo()[4]; }
    bool fading() const { return geo()[5] != 0; }
    Frames process(const Frames& input) override {
        const Index L = hop(), C = channels();
        if (input.rows() != L) throw InvalidSizeError("process() expects exactly one hop of input per call");
        if (input.cols() != C) throw InvalidInputError("input channel count does not match the filter");
        std::vector<float> in((size_t)(L * C)), out((size_t)(L * C));
        for (Index c = 0; c < C; ++c)
            for (Index t = 0; t < L; ++t) in[(size_t)(c * L + t)] = (float)input(t, c);
        check(tvolap_cmp_process_hops(h_.get(), in.data(), L, out.data(), L, 1));
        Frames y(L, C);
        for (Index c = 0; c < C; ++c)
            for (Index t = 0; t < L; ++t) y(t, c) = out[(size_t)(c * L + t)];
        return y;
    }
    void set_filter(const ImpulseResponse& ir) override {
        const std::vector<float> t = detail::channel_major(ir);
        check(tvolap_cmp_set_filter(h_.get(), t.data(), ir.length(), ir.channels(), ir.length()));
    }
    void reset() override { check(tvolap_cmp_reset(h_.get())); }

protected:
    std::vector<long> geo() const {
        std::vector<long> g(6);
        check(tvolap_cmp_geometry(h_.get(), g.data()));
        return g;
    }
    std::string name_;
    std::unique_ptr<tvolap_cmp, detail::CmpDel> h_;
};

class DirectProcessor : public CmpProcessor {  // reference.hpp:53-77
public:
    DirectProcessor(const ImpulseResponse& ir, Index hop, int device = 0)
        : CmpProcessor(TVOLAP_CMP_TDC, "tdc", ir, hop, CrossfadeConfig{}, device) {}
};

class CfTdcProcessor : public CmpProcessor {  // reference.hpp:79-118
public:
    CfTdcProcessor(const ImpulseResponse& ir, Index hop, CrossfadeConfig fade, int device = 0)
        : CmpProcessor(TVOLAP_CMP_CF_TDC, "cf-tdc", ir, hop, fade, device) {}
    void switch_filter(const ImpulseResponse& ir, const CrossfadeConfig& fade) {
        const std::vector<float> t = detail::channel_major(ir);
        check(tvolap_cmp_switch_filter(h_.get(), t.data(), ir.length(), ir.channels(), ir.length(), fade.duration,
                                       (int)fade.shape));
    }
};

class OlaProcessor : public CmpProcessor {  // reference.hpp:120-145
public:
    explicit OlaProcessor(const ImpulseResponse& ir, int device = 0)
        : CmpProcessor(TVOLAP_CMP_OLA, "ola", ir, 0, CrossfadeConfig{}, device) {}
};

class OlsProcessor : public CmpProcessor {  // reference.hpp:147-173
public:
    explicit OlsProcessor(const ImpulseResponse& ir, int device = 0)
        : CmpProcessor(TVOLAP_CMP_OLS, "ols", ir, 0, CrossfadeConfig{}, device) {}
};

class WolaProcessor : public CmpProcessor {  // reference.hpp:175-200
public:
    explicit WolaProcessor(const ImpulseResponse& ir, int device = 0)
        : CmpProcessor(TVOLAP_CMP_WOLA, "wola", ir, 0, CrossfadeConfig{}, device) {}
};

// reference.hpp:202-221
class TvolapProcessor : public StreamingProcessor {
public:
    TvolapProcessor(const ImpulseResponse& ir, Index hop, int device = 0)
        : engine_(std::make_shared<FilterPartitionSet>(partition(ir, hop, 1, device))) {}
    std::string name() const override { return "tvolap"; }
    Index hop() const override { return engine_.hop(); }
    Index channels() const override { return engine_.channels(); }
    Index latency() const override { return engine_.latency(); }
    Index stream_delay() const override { return engine_.stream_delay(); }
    Index switching_latency() const override { return engine_.switching_latency(); }
    Frames process(const Frames& input) override { return engine_.process(input); }
    void set_filter(const ImpulseResponse& ir) override {  // reference.cpp:335-338
        // validation / M as partition() (partition.cpp:21-24), the transform on the device side stream
        if (ir.length() < 1 || ir.channels() < 1) throw InvalidInputError("partition: impulse response is empty");
        auto s = std::make_shared<FilterPartitionSet>();
        s->hop = engine_.hop();
        s->partition_count = std::max((ir.length() + 2 * s->hop - 1) / (2 * s->hop), engine_.partition_count());
        s->channels = ir.channels();
        s->source_length = ir.length();
        s->sample_rate = ir.sample_rate;
        s->taps.resize((size_t)(s->channels * s->source_length));
        for (Index c = 0; c < s->channels; ++c)
            for (Index n = 0; n < s->source_length; ++n)
                s->taps[(size_t)(c * s->source_length + n)] = (float)ir.samples(n, c);
        engine_.exchange_taps(std::move(s));
    }
    void reset() override { engine_.reset(); }
    TvolapEngine& engine() { return engine_; }

private:
    TvolapEngine engine_;
};

// C3's cross-GPU stereo mix over peer memory (tvolap_mix_group_*): construct on every rank,
// all-gather handle() (64 bytes per rank, any transport), open(all); per pass scatter() on every
// rank, a host barrier, gather(), a host barrier. world == 1 needs no open().
class MixGroup {
public:
    MixGroup(int device, int world, int rank, long ears, long capacity) {
        check(tvolap_mix_group_create(&g_, device, world, rank, ears, capacity, handle_));
        if (world == 1) check(tvolap_mix_group_open(g_, nullptr));
    }
    ~MixGroup() { tvolap_mix_group_destroy(g_); }
    MixGroup(const MixGroup&) = delete;
    MixGroup& operator=(const MixGroup&) = delete;
    const char* handle() const { return handle_; }
    void open(const char* all_handles) { check(tvolap_mix_group_open(g_, all_handles)); }
    void scatter(long sources, long samples, const float* out, long out_stride, void* stream = nullptr) {
        check(tvolap_mix_scatter(g_, sources, samples, out, out_stride, stream));
    }
    void gather(long samples, float* mix, long mix_stride, void* stream = nullptr) {
        check(tvolap_mix_gather(g_, samples, mix, mix_stride, stream));
    }

private:
    tvolap_mix_group* g_ = nullptr;
    char handle_[64] = {};
};

// reference.cpp:345-363
inline std::unique_ptr<StreamingProcessor> make_processor(const std::string& name, const ImpulseResponse& ir,
                                                          Index hop, int device = 0) {
    if (name == "tdc") return std::make_unique<DirectProcessor>(ir, hop, device);
    if (name == "cf-tdc") return std::make_unique<CfTdcProcessor>(ir, hop, CrossfadeConfig{hop}, device);
    if (name == "ola") return std::make_unique<OlaProcessor>(ir, device);
    if (name == "ols") return std::make_unique<OlsProcessor>(ir, device);
    if (name == "wola") return std::make_unique<WolaProcessor>(ir, device);
    if (name == "tvolap") return std::make_unique<TvolapProcessor>(ir, hop, device);
    throw InvalidConfigurationError("unknown algorithm: " + name);
}

}  // namespace tvolap_b200
