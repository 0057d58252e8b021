// TEST INFRASTRUCTURE ONLY — C-ABI harness around the REFERENCE's own hot path.
//
// Linked (by oracle/Makefile, target `ref`) with the reference's unmodified
// sources /root/reference/proj/src/{spectral,partition,engine}.cpp, compiled
// against the minimal Eigen stand-in in oracle/eigen_shim/ (Eigen itself is not
// on disk). Output: oracle/_ref/libtvolap_ref.so (git-ignored; it travels to the
// GPU box with the snapshot, /root/reference does not).
//
// It exports the same orc_* entry points as the restated oracle
// (oracle/tvolap_oracle.cpp) for the hot-path subset, so oracle/oracle.py can
// drive either library with the same code: tests/test_ref_pin.py checks the
// restatement against the reference itself, and bench.py's --impl reference arm
// times the reference engine (kind "reference").
//
// Nothing in the product path (paper_2310_00319_b200/) links or loads this.

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "tvolap/engine.hpp"
#include "tvolap/errors.hpp"
#include "tvolap/partition.hpp"
#include "tvolap/spectral.hpp"

namespace {

using tvolap::Index;

// Status codes — identical numbering to include/tvolap_b200.h / the oracle.
enum Status : int {
    kOk = 0,
    kInvalidSize = 1,
    kInvalidInput = 2,
    kInvalidConfiguration = 3,
    kIncompatibleFilter = 4,
    kInvalidSpectrum = 5,
};

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return kOk;
    } catch (const tvolap::InvalidSizeError& e) {
        g_last_error = e.what();
        return kInvalidSize;
    } catch (const tvolap::InvalidSpectrumError& e) {
        g_last_error = e.what();
        return kInvalidSpectrum;
    } catch (const tvolap::IncompatibleFilterError& e) {
        g_last_error = e.what();
        return kIncompatibleFilter;
    } catch (const tvolap::InvalidConfigurationError& e) {
        g_last_error = e.what();
        return kInvalidConfiguration;
    } catch (const std::exception& e) {  // InvalidInputError and anything else
        g_last_error = e.what();
        return kInvalidInput;
    }
}

struct SetHandle {
    std::shared_ptr<const tvolap::FilterPartitionSet> set;
};

// taps[c * length + n] (channel-major, as the oracle takes them) -> ImpulseResponse (taps x channels)
tvolap::ImpulseResponse make_ir(const double* taps, long length, long channels) {
    tvolap::ImpulseResponse ir;
    ir.samples = Eigen::ArrayXXd::Zero(length, channels);
    for (long c = 0; c < channels; ++c)
        for (long n = 0; n < length; ++n) ir.samples(n, c) = taps[c * length + n];
    return ir;
}

}  // namespace

extern "C" {

const char* orc_last_error() { return g_last_error.c_str(); }

int orc_is_power_of_two(long n) { return tvolap::is_power_of_two(n) ? 1 : 0; }

int orc_forward_real(long n, const double* x, double* bins) {
    return guarded([&] {
        Eigen::ArrayXd block(n);
        for (long i = 0; i < n; ++i) block[i] = x[i];
        tvolap::SpectrumFrame s = tvolap::forward_real(block);
        std::memcpy(bins, s.bins.data(), sizeof(std::complex<double>) * s.bins.size());
    });
}

int orc_inverse_real(long n, long nbins, const double* bins, double* out) {
    return guarded([&] {
        Eigen::ArrayXcd b(std::max<long>(nbins, 0));
        std::memcpy((void*)b.data(), bins, sizeof(std::complex<double>) * b.size());
        tvolap::SpectrumFrame s{std::move(b), n};
        Eigen::ArrayXd y = tvolap::inverse_real(s);
        std::memcpy(out, y.data(), sizeof(double) * y.size());
    });
}

int orc_mac(long n_acc, long n_a, long n_b, long nbins_acc, long nbins_a, long nbins_b, const double* acc,
            const double* a, const double* b, double* out) {
    return guarded([&] {
        auto frame = [](const double* p, long nb, long n) {
            Eigen::ArrayXcd v(nb);
            std::memcpy((void*)v.data(), p, sizeof(std::complex<double>) * nb);
            return tvolap::SpectrumFrame{std::move(v), n};
        };
        tvolap::SpectrumFrame sa = frame(acc, nbins_acc, n_acc), x = frame(a, nbins_a, n_a),
                              y = frame(b, nbins_b, n_b);
        tvolap::mac_in_place(sa, x, y);
        std::memcpy(out, sa.bins.data(), sizeof(std::complex<double>) * nbins_acc);
    });
}

int orc_hann_window(long hop, double* w) {
    return guarded([&] {
        Eigen::ArrayXd v = tvolap::hann_window(hop);
        std::memcpy(w, v.data(), sizeof(double) * v.size());
    });
}

void* orc_partition(const double* ir, long length, long channels, long hop, long min_partitions, int* status) {
    SetHandle* h = nullptr;
    *status = guarded([&] {
        auto set = std::make_shared<const tvolap::FilterPartitionSet>(
            tvolap::partition(make_ir(ir, length, channels), hop, min_partitions));
        h = new SetHandle{std::move(set)};
    });
    return h;
}

void orc_set_free(void* s) { delete static_cast<SetHandle*>(s); }
long orc_set_partition_count(void* s) { return static_cast<SetHandle*>(s)->set->partition_count; }
long orc_set_channels(void* s) { return static_cast<SetHandle*>(s)->set->channels; }
long orc_set_hop(void* s) { return static_cast<SetHandle*>(s)->set->hop; }
long orc_set_source_length(void* s) { return static_cast<SetHandle*>(s)->set->source_length; }
double orc_set_gain(void* s) { return static_cast<SetHandle*>(s)->set->normalization_gain; }

void orc_set_spectra(void* s, double* out) {
    const auto& f = *static_cast<SetHandle*>(s)->set;
    const long nb = 2 * f.hop + 1;
    for (long c = 0; c < f.channels; ++c)
        for (long m = 0; m < f.partition_count; ++m)
            std::memcpy(out + ((c * f.partition_count + m) * nb) * 2,
                        f.partitions[static_cast<std::size_t>(c)][static_cast<std::size_t>(m)].bins.data(),
                        sizeof(std::complex<double>) * nb);
}

int orc_reassemble(void* s, double* out) {
    return guarded([&] {
        const auto& f = *static_cast<SetHandle*>(s)->set;
        tvolap::ImpulseResponse ir = tvolap::reassemble(f);
        for (long c = 0; c < ir.channels(); ++c)
            for (long n = 0; n < ir.length(); ++n) out[c * ir.length() + n] = ir.samples(n, c);
    });
}

void* orc_engine_create(void* set, int* status) {
    tvolap::TvolapEngine* e = nullptr;
    *status = guarded([&] {
        auto sp = set ? static_cast<SetHandle*>(set)->set : std::shared_ptr<const tvolap::FilterPartitionSet>{};
        e = new tvolap::TvolapEngine(sp);
    });
    return e;
}

void orc_engine_free(void* e) { delete static_cast<tvolap::TvolapEngine*>(e); }

// in[c * in_stride + n] for n < rows (channel-major, the oracle's layout): viewed, not copied, as a
// rows x cols column-major block with outer stride in_stride (an Eigen::Ref<const ArrayXXd>).
int orc_engine_process(void* e, const double* in, long in_stride, long rows, long cols, double* out,
                       long out_stride) {
    return guarded([&] {
        static const double kNone = 0.0;
        Eigen::Ref<const Eigen::ArrayXXd> view(in ? in : &kNone, rows, cols, in_stride);
        Eigen::ArrayXXd y = static_cast<tvolap::TvolapEngine*>(e)->process(view);
        for (long c = 0; c < y.cols(); ++c)
            for (long n = 0; n < y.rows(); ++n) out[c * out_stride + n] = y(n, c);
    });
}

int orc_engine_exchange(void* e, void* set) {
    return guarded([&] {
        static_cast<tvolap::TvolapEngine*>(e)->exchange_filter(
            set ? static_cast<SetHandle*>(set)->set : std::shared_ptr<const tvolap::FilterPartitionSet>{});
    });
}

void orc_engine_reset(void* e) { static_cast<tvolap::TvolapEngine*>(e)->reset(); }

void orc_engine_geometry(void* e, long* out7) {
    auto* g = static_cast<tvolap::TvolapEngine*>(e);
    out7[0] = g->hop();
    out7[1] = g->channels();
    out7[2] = g->partition_count();
    out7[3] = g->delay_line_depth();
    out7[4] = g->latency();
    out7[5] = g->switching_latency();
    out7[6] = g->stream_delay();
}

void orc_engine_op_counts(void* e, std::uint64_t* out3) {
    const auto& c = static_cast<tvolap::TvolapEngine*>(e)->op_counts();
    out3[0] = c.forward_transforms;
    out3[1] = c.inverse_transforms;
    out3[2] = c.spectral_macs;
}

// Same contract as the oracle's orc_run_workload (oracle/tvolap_oracle.cpp): the reference's
// drive() loop (proj/src/experiment.cpp:33-54) per source, run by the REFERENCE engine — stage the
// filter change right before process(); fresh IRs are partitioned at switch time on the worker
// thread as TvolapProcessor::set_filter does (reference.cpp:335-338); bank entries are
// pre-partitioned and exchanged zero-copy (engine.hpp:55). Lanes are partitioned over `threads`
// std::threads. Timed region: the threaded process/partition loop (steady_clock).
double orc_run_workload(long hop, long min_partitions, long sources, long ears, long n_hops, const double* in,
                        long in_stride, int mode, const double* fresh_ir, long ir_len, long period,
                        long n_bank, const double* bank_ir, const int* schedule, double* out, long out_stride,
                        int threads, int* status) {
    using SetPtr = std::shared_ptr<const tvolap::FilterPartitionSet>;
    *status = kOk;
    if (threads < 1) threads = 1;
    std::vector<SetPtr> bank;
    if (mode == 1) {
        bank.resize(static_cast<std::size_t>(n_bank));
        for (long b = 0; b < n_bank; ++b)
            bank[static_cast<std::size_t>(b)] = std::make_shared<const tvolap::FilterPartitionSet>(
                tvolap::partition(make_ir(bank_ir + b * ears * ir_len, ir_len, ears), hop, min_partitions));
    }
    std::atomic<int> err{kOk};
    auto worker = [&](long s0, long s1) {
        int rc = guarded([&] {
            Eigen::ArrayXXd xin(hop, ears);
            for (long s = s0; s < s1; ++s) {
                SetPtr first;
                if (mode == 0)
                    first = std::make_shared<const tvolap::FilterPartitionSet>(tvolap::partition(
                        make_ir(fresh_ir + (0 * sources + s) * ears * ir_len, ir_len, ears), hop, min_partitions));
                else
                    first = bank[static_cast<std::size_t>(schedule[s])];
                tvolap::TvolapEngine eng(first);
                int current = mode == 1 ? schedule[s] : 0;
                for (long l = 0; l < n_hops; ++l) {
                    if (mode == 0 && l > 0 && l % period == 0) {
                        const long k = l / period;
                        eng.exchange_filter(std::make_shared<const tvolap::FilterPartitionSet>(tvolap::partition(
                            make_ir(fresh_ir + (k * sources + s) * ears * ir_len, ir_len, ears), hop,
                            eng.partition_count())));
                    } else if (mode == 1 && l > 0) {
                        const int want = schedule[l * sources + s];
                        if (want != current) {
                            eng.exchange_filter(bank[static_cast<std::size_t>(want)]);
                            current = want;
                        }
                    }
                    for (long e = 0; e < ears; ++e)
                        std::memcpy(&xin(0, e), in + s * in_stride + l * hop, sizeof(double) * hop);
                    Eigen::ArrayXXd y = eng.process(xin);
                    if (out)
                        for (long e = 0; e < ears; ++e)
                            std::memcpy(out + (s * ears + e) * out_stride + l * hop, &y(0, e), sizeof(double) * hop);
                }
            }
        });
        if (rc) err = rc;
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

}  // extern "C"
