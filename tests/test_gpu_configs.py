"""GPU parity on the BASELINE.json configs: same seeded inputs/IRs into the CUDA
engine (C-ABI) and the fp64 oracle; max|y_gpu - y_ref| <= 1e-4 max|y_ref|
(north_star tolerance), across IR switches. Oracle legs run on lane subsets /
hop prefixes sized to finish in seconds (each still spans >= 2(2M-1) hops where
the ring must wrap); the GPU always runs the config's full lane count unless
noted."""
import numpy as np
import pytest

from paper_2310_00319_b200 import drive
from paper_2310_00319_b200 import workload as W
from parity import TOL, oracle_config, rel_err

pytestmark = pytest.mark.gpu


def check(cfg, n_hops, sources=None, subset=None):
    _, y = drive.run_host(cfg, n_hops, sources=sources)
    subset = list(range(sources or cfg.sources)) if subset is None else subset
    ref = oracle_config(cfg, n_hops, sources=sources, subset=subset)
    rows = [s * cfg.ears + e for s in subset for e in range(cfg.ears)]
    err = rel_err(y[rows], ref)
    assert err <= TOL, f"{cfg.name}: rel err {err:.3g}"
    return y, ref


def test_c1_full_ten_seconds():
    """C1: 1 lane, L=128, M=32, two IRs alternating every 64 blocks, all 3750 hops."""
    cfg = W.CONFIGS["C1"]
    check(cfg, cfg.hops)


def test_c2_all_lanes_fresh_switches():
    """C2: 64 lanes, L=256, M=64, fresh IR every 16 blocks; 160 hops (10 switches, ring wrapped)."""
    cfg = W.CONFIGS["C2"]
    check(cfg, 160)


def test_c3_binaural_bank():
    """C3: 1024 sources x 2 ears on the GPU (bank pass); per-block bank choice; 64 strided sources
    checked over 520 hops (ring of 255 slots wrapped)."""
    cfg = W.CONFIGS["C3"]
    subset = list(range(0, 1024, 16))
    y, ref = check(cfg, 520, subset=subset)


def test_c4_long_reverb():
    """C4: L=512, M=256, fresh IR every 8 blocks; 8 lanes over 1100 hops (ring wrapped)."""
    cfg = W.CONFIGS["C4"]
    check(cfg, 1100, sources=8)


def test_c4_full_lane_count_prefix():
    """C4 with all 256 lanes: 24 hops (3 switches), 8 strided lanes against the oracle."""
    cfg = W.CONFIGS["C4"]
    check(cfg, 24, subset=list(range(0, 256, 32)))


def test_c5_low_latency_bank():
    """C5: 4096 lanes, L=32, M=512, per-block choice from 1024 IRs (bank pass); 2100 hops (ring of
    1023 slots wrapped twice), 64 strided lanes checked."""
    cfg = W.CONFIGS["C5"]
    check(cfg, 2100, subset=list(range(0, 4096, 64)))


def test_c3_stereo_mix_against_reference_mix():
    """C3's stereo mix (tvolap_mix_allreduce, the bench path) against the fp64 sum of the reference
    outputs of ALL 1024 sources x 2 ears, over 64 hops."""
    import ctypes

    import torch

    from paper_2310_00319_b200 import tvolap as T

    cfg = W.CONFIGS["C3"]
    n, L, S = 64, cfg.hop, cfg.sources
    eng = drive.make_engine(cfg)
    x = torch.from_numpy(W.white(cfg, 0, S, 0, n * L)).cuda()
    out = torch.empty((S * cfg.ears, n * L), device="cuda")
    eng.process_hops(x, out=out, schedule=torch.from_numpy(W.schedule(cfg, 0, n)).cuda())
    mix = torch.empty((cfg.ears, n * L), device="cuda")
    eng.synchronize()
    T._check(T.lib().tvolap_mix_allreduce(0, S, cfg.ears, n * L, ctypes.c_void_p(out.data_ptr()), n * L,
                                          ctypes.c_void_p(mix.data_ptr()), n * L, None, None))
    torch.cuda.synchronize()
    ref = oracle_config(cfg, n).reshape(S, cfg.ears, -1).sum(0)
    assert rel_err(mix.cpu().numpy(), ref) <= TOL


def test_c2_full_pass_against_reference():
    """The whole 30-s C2 pass as the bench runs it (one process_switching call on device buffers,
    5625 hops, 352 fresh-IR switches) against the reference on 4 strided lanes."""
    import torch

    cfg = W.CONFIGS["C2"]
    n, L, S = cfg.hops, cfg.hop, cfg.sources
    eng = drive.make_engine(cfg)
    x = torch.from_numpy(W.white(cfg, 0, S, 0, n * L)).cuda()
    irs = [None] + _c2_device_irs(cfg, range(1, -(-n // cfg.period)), S)
    torch.cuda.synchronize()
    y = eng.process_switching(x, irs, cfg.period)
    eng.synchronize()
    subset = [0, 21, 42, 63]
    ref = oracle_config(cfg, n, subset=subset)
    assert rel_err(y.cpu().numpy()[subset], ref) <= TOL


def test_c3_mix_kernel_deterministic():
    """C3 stereo mix: device reduction over sources == fp64 sum of per-source outputs."""
    import torch

    from paper_2310_00319_b200 import tvolap as T

    cfg = W.CONFIGS["C3"]
    n_hops = 40
    eng = drive.make_engine(cfg)
    L = cfg.hop
    x = torch.from_numpy(W.white(cfg, 0, cfg.sources, 0, n_hops * L)).cuda()
    out = torch.empty((cfg.lanes, n_hops * L), device="cuda")
    sched = torch.from_numpy(W.schedule(cfg, 0, n_hops)).cuda()
    eng.process_hops(x, out=out, schedule=sched)
    eng.synchronize()
    mix = torch.empty((cfg.ears, n_hops * L), device="cuda")
    import ctypes

    rc = T.lib().tvolap_mix_device(0, cfg.sources, cfg.ears, n_hops * L, ctypes.c_void_p(out.data_ptr()),
                                   n_hops * L, ctypes.c_void_p(mix.data_ptr()), n_hops * L, None)
    assert rc == 0
    torch.cuda.synchronize()
    ref = out.double().view(cfg.sources, cfg.ears, -1).sum(0)
    assert (mix.double() - ref).abs().max().item() <= 1e-5 * ref.abs().max().item()
    mix2 = torch.empty_like(mix)
    T.lib().tvolap_mix_device(0, cfg.sources, cfg.ears, n_hops * L, ctypes.c_void_p(out.data_ptr()), n_hops * L,
                              ctypes.c_void_p(mix2.data_ptr()), n_hops * L, None)
    torch.cuda.synchronize()
    assert torch.equal(mix, mix2)


def test_device_buffers_match_host_path():
    """Device-resident (torch) process_hops == host pipeline, bit for bit (C2 prefix)."""
    import torch

    cfg = W.CONFIGS["C2"]
    n = 48
    _, y_host = drive.run_host(cfg, n)
    eng = drive.make_engine(cfg)
    x = torch.from_numpy(W.white(cfg, 0, cfg.sources, 0, n * cfg.hop)).cuda()
    out = torch.empty_like(x)
    for h0 in range(0, n, cfg.period):
        k = h0 // cfg.period
        if k:
            ir = torch.from_numpy(np.ascontiguousarray(W.fresh_irs(cfg, k)[:, 0, :])).cuda()
            eng.exchange_ir(ir)
        sl = slice(h0 * cfg.hop, (h0 + cfg.period) * cfg.hop)
        eng.process_hops(x[:, sl], out=out[:, sl])
    eng.synchronize()
    assert np.array_equal(out.cpu().numpy(), y_host)


def test_device_generators_match_host():
    """Device twins of the workload generators reproduce the host values (fp32, <= 1 ulp for IRs)."""
    import ctypes

    import torch

    from paper_2310_00319_b200 import tvolap as T

    cfg = W.CONFIGS["C2"]
    d = torch.empty((3, 1000), device="cuda")
    assert T.lib().tvolap_gen_white_device(0, cfg.seed, 5, 3, 77, 1000, ctypes.c_void_p(d.data_ptr()), 1000) == 0
    assert np.array_equal(d.cpu().numpy(), W.white(cfg, 5, 3, 77, 1000))
    items = [(3, 0, 2), (60, 0, 7)]
    host = W.ir_items(cfg, items)
    lanes = np.array([i[0] for i in items], np.int64)
    ears = np.array([i[1] for i in items], np.int64)
    ks = np.array([i[2] for i in items], np.int64)
    t60 = np.array([W.t60_of(cfg, l, k) for l, _, k in items])
    dev = torch.empty((2, cfg.ir_length), device="cuda")
    assert T.lib().tvolap_gen_irs_device(0, cfg.seed, 2, lanes.ctypes.data, ears.ctypes.data, ks.ctypes.data,
                                         t60.ctypes.data, W.FS, cfg.ir_length, ctypes.c_void_p(dev.data_ptr())) == 0
    torch.cuda.synchronize()
    assert np.abs(dev.cpu().numpy() - host).max() <= np.abs(host).max() * 2 ** -22


def _c2_device_irs(cfg, ks, S):
    """Device tensors (S, taps) of C2's fresh IR sets for switches ks (host generator)."""
    import torch

    return [torch.from_numpy(np.ascontiguousarray(W.fresh_irs(cfg, k, 0, S)[:, 0, :])).cuda() for k in ks]


def test_c2_bench_path_matches_oracle():
    """The bench's C2 path — one process_switching call on device buffers (time-parallel pass:
    K4 fused into the per-period MAC CTAs, warp-per-frame K1/K5) — over all 64 lanes and the first
    512 hops (32 fresh-IR switches, ring wrapped), 8 lanes against the fp64 oracle."""
    import torch

    cfg = W.CONFIGS["C2"]
    n, L, S = 512, cfg.hop, cfg.sources
    eng = drive.make_engine(cfg)
    x = torch.from_numpy(W.white(cfg, 0, S, 0, n * L)).cuda()
    irs = [None] + _c2_device_irs(cfg, range(1, n // cfg.period), S)
    y = eng.process_switching(x, irs, cfg.period)
    eng.synchronize()
    assert eng.wide_passes() >= 1
    subset = list(range(0, S, 8))
    ref = oracle_config(cfg, n, subset=subset)
    err = rel_err(y.cpu().numpy()[subset], ref)
    assert err <= TOL, err


def test_c2_full_pass_exact_scaling():
    """Full-size C2 pass (5625 hops x 64 lanes, 352 switches cycling 8 seeded sets): every stage is
    linear in the input and doubling is exact in fp32, so y(2x) == 2 y(x) bit for bit; outputs
    finite and nonzero; a second call from a reset engine reproduces the first exactly."""
    import torch

    cfg = W.CONFIGS["C2"]
    n, L, S = cfg.hops, cfg.hop, cfg.sources
    pool = _c2_device_irs(cfg, range(8), S)
    # every period names its set (reset() keeps the latched filter, as the reference's does)
    irs = [pool[k % 8] for k in range(-(-n // cfg.period))]
    x = torch.from_numpy(W.white(cfg, 0, S, 0, n * L)).cuda()
    x2 = 2 * x
    torch.cuda.synchronize()  # the engine runs on its own stream: inputs complete before the calls
    eng = drive.make_engine(cfg)
    y1 = eng.process_switching(x, irs, cfg.period)
    eng.reset()
    y2 = eng.process_switching(x2, irs, cfg.period)
    eng.reset()
    y3 = eng.process_switching(x, irs, cfg.period)
    eng.synchronize()
    assert eng.wide_passes() >= 3
    assert torch.isfinite(y1).all() and y1.abs().max().item() > 0
    assert torch.equal(y2, 2 * y1)
    assert torch.equal(y3, y1)


def test_c1_device_path_matches_oracle():
    """C1 on device buffers (bench path: bank schedule alternating every 64 hops -> time-parallel
    passes), all 3750 hops against the fp64 oracle."""
    import torch

    cfg = W.CONFIGS["C1"]
    n, L = cfg.hops, cfg.hop
    eng = drive.make_engine(cfg)
    x = torch.from_numpy(W.white(cfg, 0, cfg.sources, 0, n * L)).cuda()
    sched = torch.from_numpy(W.schedule(cfg, 0, n)).cuda()
    torch.cuda.synchronize()
    y = eng.process_hops(x, schedule=sched)
    eng.synchronize()
    assert eng.wide_passes() >= 1
    ref = oracle_config(cfg, n)
    assert rel_err(y.cpu().numpy(), ref) <= TOL


def test_c3_mix_allreduce_single_rank_nccl():
    """tvolap_mix_allreduce through a real (1-rank) NCCL communicator made by the C-ABI helpers:
    the all-reduce of one partial mix is that mix; NULL comm = the single-GPU mix."""
    import ctypes

    import torch

    from paper_2310_00319_b200 import tvolap as T

    cfg = W.CONFIGS["C3"]
    n_hops, S = 24, 64
    L = cfg.hop
    eng = drive.make_engine(cfg, sources=S)
    x = torch.from_numpy(W.white(cfg, 0, S, 0, n_hops * L)).cuda()
    out = torch.empty((S * cfg.ears, n_hops * L), device="cuda")
    eng.process_hops(x, out=out, schedule=torch.from_numpy(W.schedule(cfg, 0, n_hops, 0, S)).cuda())
    eng.synchronize()
    lib = T.lib()
    ref = torch.empty((cfg.ears, n_hops * L), device="cuda")
    T._check(lib.tvolap_mix_allreduce(0, S, cfg.ears, n_hops * L, ctypes.c_void_p(out.data_ptr()), n_hops * L,
                                      ctypes.c_void_p(ref.data_ptr()), n_hops * L, None, None))
    uid = (ctypes.c_char * 128)()
    T._check(lib.tvolap_nccl_unique_id(uid))
    comm = ctypes.c_void_p()
    T._check(lib.tvolap_nccl_comm_init(ctypes.byref(comm), 0, 1, 0, uid))
    got = torch.empty_like(ref)
    T._check(lib.tvolap_mix_allreduce(0, S, cfg.ears, n_hops * L, ctypes.c_void_p(out.data_ptr()), n_hops * L,
                                      ctypes.c_void_p(got.data_ptr()), n_hops * L, comm, None))
    torch.cuda.synchronize()
    T._check(lib.tvolap_nccl_comm_destroy(comm))
    assert torch.equal(got, ref)
    sums = out.double().view(S, cfg.ears, -1).sum(0)
    assert (ref.double() - sums).abs().max().item() <= 1e-5 * sums.abs().max().item()
