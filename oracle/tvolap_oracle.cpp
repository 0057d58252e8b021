// TEST INFRASTRUCTURE ONLY — the CPU oracle for the TVOLAP hot path.
//
// A plain-C++ (no Eigen), fp64 restatement of the reference engine, used by
// tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs as the checker and the CPU baseline. Nothing in the product
// path (paper_2310_00319_b200/) links, loads or calls this file.
//
// The reference (/root/reference/proj) cannot be compiled here: it needs
// Eigen3 (proj/CMakeLists.txt:12), which is not on disk, so this file restates
// the algorithm line by line:
//   * FFT tables, radix-2 DIT, real packing ........ proj/src/spectral.cpp:20-125
//   * inverse_real (tangle, 1/nc scale, checks) ..... proj/src/spectral.cpp:127-158
//   * mac_in_place (acc += a*b per bin) ............. proj/src/spectral.cpp:160-166
//   * hann_window (periodic, peak 2) ................ proj/src/partition.cpp:10-18
//   * partition / reassemble ........................ proj/src/partition.cpp:20-65
//   * TvolapEngine ctor / exchange / latch / process / reset
//                                                    proj/src/engine.cpp:9-118
//   * direct_convolve (brute force truth) ........... proj/src/reference.cpp:10-32
//   * comparison convolvers: DirectProcessor "tdc",
//     CfTdcProcessor "cf-tdc", OlaProcessor "ola", OlsProcessor "ols",
//     WolaProcessor "wola" ............................ proj/src/reference.cpp:34-320
// Parity is pinned by porting the reference's known-answer and property tests
// (proj/tests/test_spectral.cpp, test_partition.cpp, test_engine.cpp,
// acceptance.cpp crit 2-4) in tests/test_oracle.py — the reference ships no
// stored golden vectors.
//
// Exceptions of the reference become integer status codes (see
// include/tvolap_b200.h for the shared numbering) plus a thread-local message.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

namespace {

using cd = std::complex<double>;
using Index = long;

constexpr double kPi = 3.14159265358979323846264338327950288;

// Status codes — identical numbering to include/tvolap_b200.h.
enum Status : int {
    kOk = 0,
    kInvalidSize = 1,           // tvolap::InvalidSizeError
    kInvalidInput = 2,          // tvolap::InvalidInputError
    kInvalidConfiguration = 3,  // tvolap::InvalidConfigurationError
    kIncompatibleFilter = 4,    // tvolap::IncompatibleFilterError
    kInvalidSpectrum = 5,       // tvolap::InvalidSpectrumError
    kSwitchInProgress = 7,      // tvolap::SwitchInProgressError
};

struct Error {
    int code;
    std::string what;
};

thread_local std::string g_last_error;

int fail(const Error& e) {
    g_last_error = e.what;
    return e.code;
}

bool is_power_of_two(Index n) { return n > 0 && (n & (n - 1)) == 0; }

// ---------------------------------------------------------------- spectral
// spectral.cpp:22-27 — per-size tables.
struct FftTables {
    Index n_complex = 0;
    std::vector<Index> bit_reverse;
    std::vector<cd> twiddle;  // e^{-2 pi i j / nc}, j < nc/2
    std::vector<cd> pack;     // e^{-2 pi i k / (2 nc)}, k <= nc
};

// spectral.cpp:29-66 — built once per size under a mutex.
const FftTables& tables_for(Index nc) {
    static std::mutex mutex;
    static std::map<Index, std::unique_ptr<const FftTables>> cache;
    std::scoped_lock lock(mutex);
    auto it = cache.find(nc);
    if (it == cache.end()) {
        auto t = std::make_unique<FftTables>();
        t->n_complex = nc;
        int bits = 0;
        while ((Index{1} << bits) < nc) ++bits;
        t->bit_reverse.resize(nc);
        for (Index i = 0; i < nc; ++i) {
            Index r = 0;
            for (int b = 0; b < bits; ++b) r |= ((i >> b) & 1) << (bits - 1 - b);
            t->bit_reverse[i] = r;
        }
        t->twiddle.resize(nc / 2);
        for (Index j = 0; j < nc / 2; ++j) {
            const double a = -2.0 * kPi * double(j) / double(nc);
            t->twiddle[j] = {std::cos(a), std::sin(a)};
        }
        t->pack.resize(nc + 1);
        for (Index k = 0; k <= nc; ++k) {
            const double a = -2.0 * kPi * double(k) / double(2 * nc);
            t->pack[k] = {std::cos(a), std::sin(a)};
        }
        it = cache.emplace(nc, std::move(t)).first;
    }
    return *it->second;
}

inline cd cmul(cd a, cd b) {
    // Explicit form, as Eigen's packet complex product evaluates it.
    return {a.real() * b.real() - a.imag() * b.imag(), a.real() * b.imag() + a.imag() * b.real()};
}

// spectral.cpp:69-91 — iterative radix-2 DIT.
void fft_in_place(std::vector<cd>& a, const FftTables& t, bool inverse) {
    const Index n = t.n_complex;
    for (Index i = 0; i < n; ++i) {
        const Index j = t.bit_reverse[i];
        if (j > i) std::swap(a[i], a[j]);
    }
    for (Index len = 2; len <= n; len <<= 1) {
        const Index stride = n / len;
        const Index half = len / 2;
        for (Index base = 0; base < n; base += len) {
            for (Index k = 0; k < half; ++k) {
                cd w = t.twiddle[k * stride];
                if (inverse) w = std::conj(w);
                const cd u = a[base + k];
                const cd v = cmul(a[base + k + half], w);
                a[base + k] = u + v;
                a[base + k + half] = u - v;
            }
        }
    }
}

struct Spectrum {
    std::vector<cd> bins;  // n/2 + 1
    Index n = 0;           // transform length
    static Spectrum zero(Index n) { return {std::vector<cd>(n / 2 + 1), n}; }
};

// spectral.cpp:99-125
Spectrum forward_real(const double* block, Index n) {
    if (n < 8 || !is_power_of_two(n))
        throw Error{kInvalidSize, "forward_real: block length must be a power of two >= 8, got " +
                                      std::to_string(n)};
    const Index nc = n / 2;
    const FftTables& t = tables_for(nc);
    std::vector<cd> z(nc);
    for (Index j = 0; j < nc; ++j) z[j] = {block[2 * j], block[2 * j + 1]};
    fft_in_place(z, t, false);
    Spectrum s{std::vector<cd>(nc + 1), n};
    for (Index k = 0; k <= nc; ++k) {
        const cd zk = z[k % nc];
        const cd zm = std::conj(z[(nc - k) % nc]);
        const cd even = 0.5 * (zk + zm);
        const cd odd = cmul(cd{0.0, -0.5}, zk - zm);
        s.bins[k] = even + cmul(t.pack[k], odd);
    }
    s.bins[0] = {s.bins[0].real(), 0.0};
    s.bins[nc] = {s.bins[nc].real(), 0.0};
    return s;
}

// spectral.cpp:127-158
void inverse_real(const Spectrum& spec, double* out) {
    const Index n = spec.n;
    if (n < 8 || !is_power_of_two(n))
        throw Error{kInvalidSize, "inverse_real: transform length must be a power of two >= 8, got " +
                                      std::to_string(n)};
    const Index nc = n / 2;
    if (Index(spec.bins.size()) != nc + 1)
        throw Error{kInvalidSize, "inverse_real: expected " + std::to_string(nc + 1) + " bins, got " +
                                      std::to_string(spec.bins.size())};
    if (spec.bins[0].imag() != 0.0 || spec.bins[nc].imag() != 0.0)
        throw Error{kInvalidSpectrum, "inverse_real: DC and Nyquist bins must have zero imaginary part"};
    const FftTables& t = tables_for(nc);
    std::vector<cd> z(nc);
    for (Index k = 0; k < nc; ++k) {
        const cd xk = spec.bins[k];
        const cd xm = std::conj(spec.bins[nc - k]);
        const cd even = 0.5 * (xk + xm);
        const cd odd = cmul(0.5 * (xk - xm), std::conj(t.pack[k]));
        z[k] = even + cmul(cd{0.0, 1.0}, odd);
    }
    fft_in_place(z, t, true);
    const double scale = 1.0 / double(nc);
    for (Index j = 0; j < nc; ++j) {
        out[2 * j] = z[j].real() * scale;
        out[2 * j + 1] = z[j].imag() * scale;
    }
}

// spectral.cpp:160-166
void mac_in_place(Spectrum& acc, const Spectrum& a, const Spectrum& b) {
    if (acc.n != a.n || a.n != b.n) throw Error{kInvalidSize, "mac: transform lengths differ"};
    if (acc.bins.size() != a.bins.size() || a.bins.size() != b.bins.size())
        throw Error{kInvalidSize, "mac: bin counts differ"};
    const std::size_t nb = acc.bins.size();
    cd* __restrict__ pa = acc.bins.data();
    const cd* __restrict__ x = a.bins.data();
    const cd* __restrict__ y = b.bins.data();
    for (std::size_t k = 0; k < nb; ++k) pa[k] += cmul(x[k], y[k]);
}

// ---------------------------------------------------------------- partition
// partition.cpp:10-18
std::vector<double> hann_window(Index hop) {
    if (hop < 2) throw Error{kInvalidSize, "hann_window: hop size must be >= 2, got " + std::to_string(hop)};
    const Index n = 2 * hop;
    std::vector<double> w(n);
    for (Index i = 0; i < n; ++i) w[i] = 1.0 - std::cos(2.0 * kPi * double(i) / double(n));
    return w;
}

// partition.hpp:21-32
struct FilterSet {
    Index hop = 0;
    Index partition_count = 0;
    Index channels = 0;
    Index source_length = 0;
    double normalization_gain = 0.5;
    std::vector<std::vector<Spectrum>> partitions;  // [channel][m]
    Index transform_length() const { return 4 * hop; }
};

// partition.cpp:20-51. `ir` is channel-major: ir[c * length + i].
std::shared_ptr<const FilterSet> partition(const double* ir, Index length, Index channels, Index hop,
                                           Index min_partitions) {
    if (length < 1 || channels < 1) throw Error{kInvalidInput, "partition: impulse response is empty"};
    if (hop < 2 || !is_power_of_two(4 * hop))
        throw Error{kInvalidSize, "partition: 4L must be a power of two, got L = " + std::to_string(hop)};
    const Index slice = 2 * hop;
    const Index m = std::max((length + slice - 1) / slice, std::max<Index>(min_partitions, 1));
    auto set = std::make_shared<FilterSet>();
    set->hop = hop;
    set->partition_count = m;
    set->channels = channels;
    set->source_length = length;
    set->partitions.resize(channels);
    std::vector<double> padded(4 * hop);
    for (Index c = 0; c < channels; ++c) {
        auto& frames = set->partitions[c];
        frames.reserve(m);
        for (Index p = 0; p < m; ++p) {
            const Index begin = p * slice;
            const Index count = std::clamp<Index>(length - begin, 0, slice);
            std::fill(padded.begin(), padded.end(), 0.0);
            for (Index i = 0; i < count; ++i) padded[i] = ir[c * length + begin + i];
            frames.push_back(forward_real(padded.data(), 4 * hop));
        }
    }
    return set;
}

// ---------------------------------------------------------------- engine
// engine.hpp:17-21
struct OpCounts {
    std::uint64_t forward_transforms = 0;
    std::uint64_t inverse_transforms = 0;
    std::uint64_t spectral_macs = 0;
};

// engine.hpp:33-94 / engine.cpp:9-118
class Engine {
public:
    explicit Engine(std::shared_ptr<const FilterSet> filter) : filter_(std::move(filter)) {
        if (!filter_) throw Error{kInvalidConfiguration, "engine requires a filter partition set"};
        hop_ = filter_->hop;
        partition_count_ = filter_->partition_count;
        channels_ = filter_->channels;
        if (hop_ < 2 || partition_count_ < 1 || channels_ < 1)
            throw Error{kInvalidConfiguration, "degenerate filter partition set"};
        window_ = hann_window(hop_);
        const Index n = filter_->transform_length();
        state_.resize(channels_);
        for (auto& st : state_) {
            st.history.assign(hop_, 0.0);
            st.spectra.assign(delay_line_depth(), Spectrum::zero(n));
            st.tail_prev.assign(2 * hop_, 0.0);
            st.tail_prev2.assign(2 * hop_, 0.0);
            st.carry.assign(hop_, 0.0);
        }
        padded_.assign(n, 0.0);
        acc_ = Spectrum::zero(n);
        y_.assign(n, 0.0);
        ov_.assign(2 * hop_, 0.0);
    }

    Index hop() const { return hop_; }
    Index channels() const { return channels_; }
    Index partition_count() const { return partition_count_; }
    Index delay_line_depth() const { return 2 * partition_count_ - 1; }
    Index latency() const { return 2 * hop_; }
    Index switching_latency() const { return hop_; }
    Index stream_delay() const { return hop_; }
    const OpCounts& op_counts() const { return counts_; }

    // engine.cpp:37-48
    void exchange_filter(std::shared_ptr<const FilterSet> next) {
        if (!next) throw Error{kIncompatibleFilter, "replacement filter is null"};
        if (next->hop != hop_) throw Error{kIncompatibleFilter, "replacement filter hop differs"};
        if (next->partition_count != partition_count_)
            throw Error{kIncompatibleFilter, "replacement filter partition count differs"};
        if (next->channels != channels_)
            throw Error{kIncompatibleFilter, "replacement filter channel count differs"};
        std::lock_guard<std::mutex> lock(pending_mutex_);
        pending_ = std::move(next);
    }

    // engine.cpp:60-106. in/out are channel-major [c * in_stride + t], t < L.
    void process(const double* in, Index in_stride, Index rows, Index cols, double* out, Index out_stride) {
        latch_pending_filter();
        const Index L = hop_;
        if (rows != L) throw Error{kInvalidSize, "process() expects exactly one hop of input per call"};
        if (cols != channels_) throw Error{kInvalidInput, "input channel count does not match the filter"};
        const Index depth = delay_line_depth();
        const Index new_head = (ring_head_ + depth - 1) % depth;
        const double gain = filter_->normalization_gain;
        for (Index c = 0; c < channels_; ++c) {
            auto& st = state_[c];
            const double* x = in + c * in_stride;
            std::fill(padded_.begin(), padded_.end(), 0.0);
            for (Index i = 0; i < L; ++i) padded_[i] = st.history[i] * window_[i];
            for (Index i = 0; i < L; ++i) padded_[L + i] = x[i] * window_[L + i];
            for (Index i = 0; i < L; ++i) st.history[i] = x[i];
            st.spectra[new_head] = forward_real(padded_.data(), 4 * L);
            ++counts_.forward_transforms;

            std::fill(acc_.bins.begin(), acc_.bins.end(), cd{});
            const auto& parts = filter_->partitions[c];
            for (Index m = 0; m < partition_count_; ++m) {
                const Index slot = (new_head + 2 * m) % depth;
                mac_in_place(acc_, parts[m], st.spectra[slot]);
                ++counts_.spectral_macs;
            }
            inverse_real(acc_, y_.data());
            ++counts_.inverse_transforms;

            double* o = out + c * out_stride;
            for (Index i = 0; i < 2 * L; ++i) ov_[i] = y_[i] + st.tail_prev2[i];
            for (Index i = 0; i < L; ++i) o[i] = gain * (ov_[i] + st.carry[i]);
            for (Index i = 0; i < L; ++i) st.carry[i] = ov_[L + i];
            std::swap(st.tail_prev2, st.tail_prev);
            for (Index i = 0; i < 2 * L; ++i) st.tail_prev[i] = y_[2 * L + i];
        }
        ring_head_ = new_head;
    }

    // engine.cpp:108-118
    void reset() {
        for (auto& st : state_) {
            std::fill(st.history.begin(), st.history.end(), 0.0);
            for (auto& f : st.spectra) std::fill(f.bins.begin(), f.bins.end(), cd{});
            std::fill(st.tail_prev.begin(), st.tail_prev.end(), 0.0);
            std::fill(st.tail_prev2.begin(), st.tail_prev2.end(), 0.0);
            std::fill(st.carry.begin(), st.carry.end(), 0.0);
        }
        ring_head_ = 0;
    }

    const FilterSet& filter() const { return *filter_; }

private:
    struct ChannelState {
        std::vector<double> history;
        std::vector<Spectrum> spectra;
        std::vector<double> tail_prev;
        std::vector<double> tail_prev2;
        std::vector<double> carry;
    };

    // engine.cpp:54-58
    void latch_pending_filter() {
        std::lock_guard<std::mutex> lock(pending_mutex_);
        if (pending_) filter_ = std::move(pending_);
    }

    Index hop_ = 0, partition_count_ = 0, channels_ = 0;
    std::shared_ptr<const FilterSet> filter_, pending_;
    std::mutex pending_mutex_;
    std::vector<double> window_;
    std::vector<ChannelState> state_;
    Index ring_head_ = 0;
    std::vector<double> padded_, y_, ov_;
    Spectrum acc_;
    OpCounts counts_;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const Error& e) {
        return fail(e);
    } catch (const std::exception& e) {
        return fail(Error{kInvalidInput, e.what()});
    }
}

struct SetHandle {
    std::shared_ptr<const FilterSet> set;
};

// ---------------------------------------------------------------- comparison convolvers
// reference.cpp:34-320. All state is channel-major; process() takes exactly hop() rows.
enum CmpKind : int { kTdc = 0, kCfTdc = 1, kOla = 2, kOls = 3, kWola = 4 };

struct Cmp {
    int kind = kTdc;
    Index hop = 0, taps = 0, channels = 0, block = 0;
    // time-domain forms (reference.cpp:57-180)
    std::vector<double> coeffs, old_coeffs, pending_coeffs, history;  // [c][taps], history [c][taps-1]
    bool pending = false;
    Index fade_duration = 1, pending_duration = 1, fade_remaining = 0, fade_elapsed = 0;
    int fade_shape = 0, pending_shape = 0;  // 0 Hann-complementary, 1 linear
    // block forms (reference.cpp:182-320)
    std::vector<Spectrum> spectra, pending_spectra;  // per channel, transform 2*block
    std::vector<double> remainder, previous, analysis, wola_hist, acc;

    Index latency() const { return kind == kOla || kind == kOls || kind == kWola ? block : 0; }
    Index stream_delay() const { return kind == kWola ? block / 2 : 0; }
    Index switching_latency() const { return kind == kCfTdc ? fade_duration : (kind == kWola ? block / 2 : 0); }

    // reference.cpp:44-55: zero-padded spectrum of each channel, transform length 2*block
    std::vector<Spectrum> block_spectra(const double* ir) const {
        std::vector<Spectrum> out;
        std::vector<double> padded(2 * block);
        for (Index c = 0; c < channels; ++c) {
            std::fill(padded.begin(), padded.end(), 0.0);
            for (Index i = 0; i < block; ++i) padded[i] = ir[c * block + i];
            out.push_back(forward_real(padded.data(), 2 * block));
        }
        return out;
    }

    // reference.cpp:110-120
    double new_gain(Index t) const {
        const Index d = fade_duration;
        if (t >= d || d == 1) return 1.0;
        const double phase = double(t) / double(d);
        if (fade_shape == 1) return phase;
        return 0.5 * (1.0 - std::cos(kPi * phase));
    }

    void check(Index rows, Index cols) const {
        if (rows != hop) throw Error{kInvalidSize, "process() expects exactly one hop of input per call"};
        if (cols != channels) throw Error{kInvalidInput, "input channel count does not match the filter"};
    }

    void set_filter(const double* ir, Index n_taps, Index n_ch) {
        if (kind == kCfTdc) return switch_filter(ir, n_taps, n_ch, fade_duration, fade_shape);
        if (n_taps != taps || n_ch != channels) throw Error{kIncompatibleFilter, "replacement filter shape differs"};
        if (kind == kTdc) {
            pending_coeffs.assign(ir, ir + taps * channels);
            pending = true;
        } else {
            pending_spectra = block_spectra(ir);
        }
    }

    // reference.cpp:122-132
    void switch_filter(const double* ir, Index n_taps, Index n_ch, Index duration, int shape) {
        if (fade_remaining > 0 || pending) throw Error{kSwitchInProgress, "a crossfade is already in progress"};
        if (n_taps != taps || n_ch != channels) throw Error{kIncompatibleFilter, "replacement filter shape differs"};
        if (duration < 1) throw Error{kInvalidConfiguration, "crossfade duration must be >= 1"};
        pending_coeffs.assign(ir, ir + taps * channels);
        pending_duration = duration;
        pending_shape = shape;
        pending = true;
    }

    // y_i = sum_q h[q] * buf[i + taps - 1 - q] (reference.cpp:87-90, 157-159)
    static double fir(const double* h, const double* buf, Index i, Index taps) {
        double s = 0.0;
        for (Index q = 0; q < taps; ++q) s += h[q] * buf[i + taps - 1 - q];
        return s;
    }

    void process(const double* in, Index in_stride, Index rows, Index cols, double* out, Index out_stride) {
        if (kind == kTdc || kind == kCfTdc) {
            if (pending) {  // reference.cpp:72-76 / 137-146
                if (kind == kCfTdc) {
                    old_coeffs.swap(coeffs);
                    fade_duration = pending_duration;
                    fade_shape = pending_shape;
                    fade_remaining = fade_duration;
                    fade_elapsed = 0;
                }
                coeffs = pending_coeffs;
                pending = false;
            }
            check(rows, cols);
            std::vector<double> buf(taps - 1 + hop);
            std::vector<Index> elapsed(hop);
            std::vector<char> blend(hop);
            for (Index i = 0; i < hop; ++i) {  // the fade clock advances per sample (reference.cpp:153-171)
                blend[i] = kind == kCfTdc && fade_remaining > 0;
                elapsed[i] = fade_elapsed;
                if (blend[i]) {
                    ++fade_elapsed;
                    --fade_remaining;
                }
            }
            for (Index c = 0; c < channels; ++c) {
                std::copy(history.begin() + c * (taps - 1), history.begin() + (c + 1) * (taps - 1), buf.begin());
                for (Index i = 0; i < hop; ++i) buf[taps - 1 + i] = in[c * in_stride + i];
                const double* h = coeffs.data() + c * taps;
                for (Index i = 0; i < hop; ++i) {
                    const double y_new = fir(h, buf.data(), i, taps);
                    if (blend[i]) {
                        const double g_new = new_gain(elapsed[i]);
                        out[c * out_stride + i] =
                            (1.0 - g_new) * fir(old_coeffs.data() + c * taps, buf.data(), i, taps) + g_new * y_new;
                    } else {
                        out[c * out_stride + i] = y_new;
                    }
                }
                std::copy(buf.begin() + hop, buf.end(), history.begin() + c * (taps - 1));
            }
            return;
        }
        if (!pending_spectra.empty()) {  // the saved tails keep whatever filter produced them
            spectra = std::move(pending_spectra);
            pending_spectra.clear();
        }
        check(rows, cols);
        const Index n = 2 * block;
        std::vector<double> frame(n), y(n);
        for (Index c = 0; c < channels; ++c) {
            const double* x = in + c * in_stride;
            double* o = out + c * out_stride;
            std::fill(frame.begin(), frame.end(), 0.0);
            if (kind == kOla) {  // reference.cpp:205-216
                for (Index i = 0; i < block; ++i) frame[i] = x[i];
            } else if (kind == kOls) {  // reference.cpp:241-252
                for (Index i = 0; i < block; ++i) frame[i] = previous[c * block + i];
                for (Index i = 0; i < block; ++i) frame[block + i] = x[i];
            } else {  // WOLA, reference.cpp:283-306
                const Index half = block / 2;
                for (Index i = 0; i < half; ++i) frame[i] = wola_hist[c * half + i] * analysis[i];
                for (Index i = 0; i < half; ++i) frame[half + i] = x[i] * analysis[half + i];
                for (Index i = 0; i < half; ++i) wola_hist[c * half + i] = x[i];
            }
            const Spectrum xs = forward_real(frame.data(), n);
            Spectrum accs = Spectrum::zero(n);
            mac_in_place(accs, xs, spectra[c]);
            inverse_real(accs, y.data());
            if (kind == kOla) {
                for (Index i = 0; i < block; ++i) o[i] = y[i] + remainder[c * block + i];
                for (Index i = 0; i < block; ++i) remainder[c * block + i] = y[block + i];
            } else if (kind == kOls) {
                for (Index i = 0; i < block; ++i) o[i] = y[block + i];  // first half carries the circular wrap
                for (Index i = 0; i < block; ++i) previous[c * block + i] = x[i];
            } else {
                const Index half = block / 2;
                for (Index i = 0; i < block; ++i) y[i] *= analysis[i];  // synthesis window over the block
                double* a = acc.data() + c * n;
                for (Index i = 0; i < n; ++i) a[i] += y[i];
                for (Index i = 0; i < half; ++i) o[i] = 0.5 * a[i];
                for (Index i = 0; i < n - half; ++i) a[i] = a[i + half];
                for (Index i = n - half; i < n; ++i) a[i] = 0.0;
            }
        }
    }

    void reset() {
        std::fill(history.begin(), history.end(), 0.0);
        fade_remaining = 0;
        fade_elapsed = 0;
        std::fill(remainder.begin(), remainder.end(), 0.0);
        std::fill(previous.begin(), previous.end(), 0.0);
        std::fill(wola_hist.begin(), wola_hist.end(), 0.0);
        std::fill(acc.begin(), acc.end(), 0.0);
    }
};

// Constructors (reference.cpp:59-66, 97-108, 184-190, 221-227, 259-267); `ir` channel-major.
Cmp* make_cmp(int kind, const double* ir, Index taps, Index channels, Index hop, Index fade_duration,
              int fade_shape) {
    auto p = std::make_unique<Cmp>();
    p->kind = kind;
    p->taps = taps;
    p->channels = channels;
    if (kind == kTdc || kind == kCfTdc) {
        if (hop < 1) throw Error{kInvalidConfiguration, "hop must be positive"};
        if (taps < 1 || channels < 1) throw Error{kInvalidInput, "empty impulse response"};
        if (kind == kCfTdc && fade_duration < 1) throw Error{kInvalidConfiguration, "crossfade duration must be >= 1"};
        p->hop = hop;
        p->coeffs.assign(ir, ir + taps * channels);
        p->old_coeffs.assign(taps * channels, 0.0);
        p->history.assign((taps - 1) * channels, 0.0);
        p->fade_duration = fade_duration;
        p->fade_shape = fade_shape;
    } else if (kind == kOla || kind == kOls || kind == kWola) {
        if (taps < 4 || !is_power_of_two(taps))
            throw Error{kInvalidSize, "block fast convolution needs a power-of-two response length >= 4"};
        if (channels < 1) throw Error{kInvalidInput, "empty impulse response"};
        p->block = taps;
        p->hop = kind == kWola ? taps / 2 : taps;
        p->spectra = p->block_spectra(ir);
        p->remainder.assign(taps * channels, 0.0);
        p->previous.assign(taps * channels, 0.0);
        if (kind == kWola) {
            p->analysis = hann_window(taps / 2);
            for (double& v : p->analysis) v = std::sqrt(v);
            p->wola_hist.assign(taps / 2 * channels, 0.0);
            p->acc.assign(2 * taps * channels, 0.0);
        }
    } else {
        throw Error{kInvalidConfiguration, "unknown algorithm"};
    }
    return p.release();
}

}  // namespace

// ======================================================================= C ABI
extern "C" {

const char* orc_last_error() { return g_last_error.c_str(); }

int orc_is_power_of_two(long n) { return is_power_of_two(n) ? 1 : 0; }

// forward_real: x[n] -> bins[(n/2+1)*2] interleaved re/im.
int orc_forward_real(long n, const double* x, double* bins) {
    return guarded([&] {
        Spectrum s = forward_real(x, n);
        std::memcpy(bins, s.bins.data(), sizeof(cd) * s.bins.size());
    });
}

// inverse_real: bins[(nbins)*2] with declared transform length n -> out[n].
int orc_inverse_real(long n, long nbins, const double* bins, double* out) {
    return guarded([&] {
        Spectrum s{std::vector<cd>(std::max<long>(nbins, 0)), n};
        std::memcpy((void*)s.bins.data(), bins, sizeof(cd) * s.bins.size());
        inverse_real(s, out);
    });
}

// mac: out = acc + a*b, all (n/2+1) complex interleaved.
int orc_mac(long n_acc, long n_a, long n_b, long nbins_acc, long nbins_a, long nbins_b, const double* acc,
            const double* a, const double* b, double* out) {
    return guarded([&] {
        Spectrum sa{std::vector<cd>(nbins_acc), n_acc}, x{std::vector<cd>(nbins_a), n_a},
            y{std::vector<cd>(nbins_b), n_b};
        std::memcpy((void*)sa.bins.data(), acc, sizeof(cd) * nbins_acc);
        std::memcpy((void*)x.bins.data(), a, sizeof(cd) * nbins_a);
        std::memcpy((void*)y.bins.data(), b, sizeof(cd) * nbins_b);
        mac_in_place(sa, x, y);
        std::memcpy(out, sa.bins.data(), sizeof(cd) * nbins_acc);
    });
}

int orc_hann_window(long hop, double* w) {
    return guarded([&] {
        auto v = hann_window(hop);
        std::memcpy(w, v.data(), sizeof(double) * v.size());
    });
}

// partition(ir, hop, min_partitions) -> opaque set handle (shared, immutable).
void* orc_partition(const double* ir, long length, long channels, long hop, long min_partitions, int* status) {
    SetHandle* h = nullptr;
    *status = guarded([&] { h = new SetHandle{partition(ir, length, channels, hop, min_partitions)}; });
    return h;
}

void orc_set_free(void* s) { delete static_cast<SetHandle*>(s); }

long orc_set_partition_count(void* s) { return static_cast<SetHandle*>(s)->set->partition_count; }
long orc_set_channels(void* s) { return static_cast<SetHandle*>(s)->set->channels; }
long orc_set_hop(void* s) { return static_cast<SetHandle*>(s)->set->hop; }
long orc_set_source_length(void* s) { return static_cast<SetHandle*>(s)->set->source_length; }
double orc_set_gain(void* s) { return static_cast<SetHandle*>(s)->set->normalization_gain; }

// Copy spectra out: out[c][m][bin][2].
void orc_set_spectra(void* s, double* out) {
    const FilterSet& f = *static_cast<SetHandle*>(s)->set;
    const long nb = 2 * f.hop + 1;
    for (long c = 0; c < f.channels; ++c)
        for (long m = 0; m < f.partition_count; ++m)
            std::memcpy(out + ((c * f.partition_count + m) * nb) * 2, f.partitions[c][m].bins.data(),
                        sizeof(cd) * nb);
}

// partition.cpp:53-65 — reassemble: out[c][M*2L].
int orc_reassemble(void* s, double* out) {
    return guarded([&] {
        const FilterSet& f = *static_cast<SetHandle*>(s)->set;
        const long slice = 2 * f.hop;
        std::vector<double> block(4 * f.hop);
        for (long c = 0; c < f.channels; ++c)
            for (long p = 0; p < f.partition_count; ++p) {
                inverse_real(f.partitions[c][p], block.data());
                std::memcpy(out + c * slice * f.partition_count + p * slice, block.data(), sizeof(double) * slice);
            }
    });
}

void* orc_engine_create(void* set, int* status) {
    Engine* e = nullptr;
    *status = guarded([&] {
        auto sp = set ? static_cast<SetHandle*>(set)->set : std::shared_ptr<const FilterSet>{};
        e = new Engine(sp);
    });
    return e;
}

void orc_engine_free(void* e) { delete static_cast<Engine*>(e); }

int orc_engine_process(void* e, const double* in, long in_stride, long rows, long cols, double* out,
                       long out_stride) {
    return guarded([&] { static_cast<Engine*>(e)->process(in, in_stride, rows, cols, out, out_stride); });
}

int orc_engine_exchange(void* e, void* set) {
    return guarded([&] {
        static_cast<Engine*>(e)->exchange_filter(set ? static_cast<SetHandle*>(set)->set
                                                     : std::shared_ptr<const FilterSet>{});
    });
}

void orc_engine_reset(void* e) { static_cast<Engine*>(e)->reset(); }

void orc_engine_geometry(void* e, long* out7) {
    auto* g = static_cast<Engine*>(e);
    out7[0] = g->hop();
    out7[1] = g->channels();
    out7[2] = g->partition_count();
    out7[3] = g->delay_line_depth();
    out7[4] = g->latency();
    out7[5] = g->switching_latency();
    out7[6] = g->stream_delay();
}

void orc_engine_op_counts(void* e, std::uint64_t* out3) {
    const auto& c = static_cast<Engine*>(e)->op_counts();
    out3[0] = c.forward_transforms;
    out3[1] = c.inverse_transforms;
    out3[2] = c.spectral_macs;
}

// reference.cpp:10-32 — single channel brute-force linear convolution.
void orc_direct_convolve(const double* x, long n, const double* h, long taps, double* out) {
    std::fill(out, out + n + taps - 1, 0.0);
    for (long q = 0; q < taps; ++q) {
        const double w = h[q];
        if (w != 0.0)
            for (long i = 0; i < n; ++i) out[q + i] += w * x[i];
    }
}

// --------------------------------------------------------------- workload driver
// Streams `n_hops` hops of a multi-lane workload through one reference engine
// per source, the way the reference's drive() loop does
// (proj/src/experiment.cpp:33-54): per hop, stage the filter change (if any)
// right before process(). Lanes are partitioned over `threads` std::threads,
// which the spec allows. Returns seconds of wall time spent in
// the threaded process/partition region (steady_clock, like the reference);
// generation of inputs and IRs happens in the caller, outside the timer.
//
// mode 0 ("fresh"):  per source s, a new time-domain IR every `period` hops,
//                    taken from fresh_ir[(k * sources + s) * ears * ir_len ...]
//                    for switch k (k = hop / period), partitioned at switch
//                    time on the worker thread (as TvolapProcessor::set_filter
//                    does, reference.cpp:335-338). The IR for hop 0 is k = 0.
// mode 1 ("bank"):   pre-partitioned bank sets (one per bank entry, ears
//                    channels), selected per (hop, source) by
//                    schedule[hop * sources + s]; exchanged zero-copy when the
//                    choice changes (engine.hpp:55).
// Input:  in[s * in_stride + t], t < n_hops * hop (ears share the source input,
//         fanned out like audio_buffer.hpp:60-67).
// Output: out[(s * ears + e) * out_stride + t] when out != nullptr.
double orc_run_workload(long hop, long min_partitions, long sources, long ears, long n_hops, const double* in,
                        long in_stride, int mode, const double* fresh_ir, long ir_len, long period,
                        long n_bank, const double* bank_ir, const int* schedule, double* out, long out_stride,
                        int threads, int* status) {
    *status = kOk;
    if (threads < 1) threads = 1;
    std::vector<std::shared_ptr<const FilterSet>> bank;
    if (mode == 1) {
        bank.resize(n_bank);
        for (long b = 0; b < n_bank; ++b)
            bank[b] = partition(bank_ir + b * ears * ir_len, ir_len, ears, hop, min_partitions);
    }
    std::atomic<int> err{kOk};
    auto worker = [&](long s0, long s1) {
        try {
            std::vector<double> xin(ears * hop), yout(ears * hop), irbuf(ears * ir_len);
            for (long s = s0; s < s1; ++s) {
                std::shared_ptr<const FilterSet> first;
                if (mode == 0) {
                    first = partition(fresh_ir + (0 * sources + s) * ears * ir_len, ir_len, ears, hop, min_partitions);
                } else {
                    first = bank[schedule[0 * sources + s]];
                }
                Engine eng(first);
                int current = mode == 1 ? schedule[s] : 0;
                for (long l = 0; l < n_hops; ++l) {
                    if (mode == 0 && l > 0 && l % period == 0) {
                        const long k = l / period;
                        eng.exchange_filter(partition(fresh_ir + (k * sources + s) * ears * ir_len, ir_len, ears,
                                                      hop, eng.partition_count()));
                    } else if (mode == 1 && l > 0) {
                        const int want = schedule[l * sources + s];
                        if (want != current) {
                            eng.exchange_filter(bank[want]);
                            current = want;
                        }
                    }
                    for (long e = 0; e < ears; ++e)
                        std::memcpy(xin.data() + e * hop, in + s * in_stride + l * hop, sizeof(double) * hop);
                    eng.process(xin.data(), hop, hop, ears, yout.data(), hop);
                    if (out)
                        for (long e = 0; e < ears; ++e)
                            std::memcpy(out + (s * ears + e) * out_stride + l * hop, yout.data() + e * hop,
                                        sizeof(double) * hop);
                }
            }
        } catch (const Error& e) {
            g_last_error = e.what;
            err = e.code;
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    const long per = (sources + threads - 1) / threads;
    for (int t = 0; t < threads; ++t) {
        const long s0 = t * per, s1 = std::min(sources, s0 + per);
        if (s0 < s1) pool.emplace_back(worker, s0, s1);
    }
    for (auto& th : pool) th.join();
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *status = err.load();
    return secs;
}


// ---- comparison convolvers; kind: 0 tdc, 1 cf-tdc, 2 ola, 3 ols, 4 wola
void* orc_cmp_create(int kind, const double* ir, long taps, long channels, long hop, long fade_duration,
                     int fade_shape, int* status) {
    Cmp* p = nullptr;
    *status = guarded([&] { p = make_cmp(kind, ir, taps, channels, hop, fade_duration, fade_shape); });
    return p;
}

void orc_cmp_free(void* p) { delete static_cast<Cmp*>(p); }

int orc_cmp_process(void* p, const double* in, long in_stride, long rows, long cols, double* out, long out_stride) {
    return guarded([&] { static_cast<Cmp*>(p)->process(in, in_stride, rows, cols, out, out_stride); });
}

int orc_cmp_set_filter(void* p, const double* ir, long taps, long channels) {
    return guarded([&] { static_cast<Cmp*>(p)->set_filter(ir, taps, channels); });
}

int orc_cmp_switch_filter(void* p, const double* ir, long taps, long channels, long duration, int shape) {
    return guarded([&] {
        auto* c = static_cast<Cmp*>(p);
        if (c->kind != kCfTdc) throw Error{kInvalidConfiguration, "switch_filter needs a cf-tdc processor"};
        c->switch_filter(ir, taps, channels, duration, shape);
    });
}

void orc_cmp_reset(void* p) { static_cast<Cmp*>(p)->reset(); }

// hop, channels, latency, stream_delay, switching_latency, fading
void orc_cmp_geometry(void* p, long* out6) {
    const auto* c = static_cast<Cmp*>(p);
    out6[0] = c->hop;
    out6[1] = c->channels;
    out6[2] = c->latency();
    out6[3] = c->stream_delay();
    out6[4] = c->switching_latency();
    out6[5] = c->fade_remaining > 0 ? 1 : 0;
}

}  // extern "C"
