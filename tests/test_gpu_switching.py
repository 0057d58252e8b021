"""tvolap_process_switching: one launch with in-kernel K4 in the barrier gaps must equal the
exchange_filter + process_hops loop it stands for, bit for bit (and the oracle within 1e-4)."""
import numpy as np
import pytest

import oracle as O
from paper_2310_00319_b200 import tvolap as T

pytestmark = pytest.mark.gpu


def _case(hop, S, taps, n_hops, period, none_at=(), seed=0):
    import torch

    g = np.random.default_rng(seed)
    nsw = -(-n_hops // period)
    irs = [None if k in none_at else g.standard_normal((S, taps)).astype(np.float32) * 0.05 for k in range(nsw)]
    ir0 = g.standard_normal((taps, S)) * 0.05
    x = torch.from_numpy(g.uniform(-1, 1, (S, n_hops * hop)).astype(np.float32)).cuda()
    dirs = [None if ir is None else torch.from_numpy(ir).cuda() for ir in irs]
    return ir0, x, dirs


def _loop(eng, x, dirs, period, hop):
    import torch

    n = x.shape[1] // hop
    out = torch.empty_like(x)
    for k in range(-(-n // period)):
        if dirs[k] is not None:
            eng.exchange_ir(dirs[k])
        sl = slice(k * period * hop, min(n, (k + 1) * period) * hop)
        eng.process_hops(x[:, sl], out=out[:, sl])
    return out


@pytest.mark.parametrize("hop,S,taps,n_hops,period,none_at", [
    (256, 5, 4096, 16 * 5 + 7, 16, (2,)),   # C2-like: one 16-hop block per period, ragged tail
    (256, 3, 3000, 61, 10, ()),             # periods shorter than a block
    (256, 3, 4096, 100, 40, (1,)),          # periods spanning several blocks
    (128, 4, 2048, 70, 16, ()),             # N = 256
    (512, 2, 8192, 48, 8, (0,)),            # N = 1024, no switch at the first hop
])
def test_switching_equals_exchange_loop(monkeypatch, hop, S, taps, n_hops, period, none_at):
    T.set_default_tuning("wide", 0)  # the hop-blocked switching launch (the pass: test_gpu_wide.py)
    ir0, x, dirs = _case(hop, S, taps, n_hops, period, none_at)
    a = T.TvolapEngine(T.partition(ir0, hop))
    b = T.TvolapEngine(T.partition(ir0, hop))
    a.process_hops(x[:, : 3 * hop])  # some history first (odd start hop)
    b.process_hops(x[:, : 3 * hop])
    ya = a.process_switching(x, dirs, period)
    yb = _loop(b, x, dirs, period, hop)
    a.synchronize()
    b.synchronize()
    assert np.array_equal(ya.cpu().numpy(), yb.cpu().numpy())
    # and the engines continue identically afterwards
    za, zb = a.process_hops(x[:, : 8 * hop]), b.process_hops(x[:, : 8 * hop])
    assert np.array_equal(za.cpu().numpy(), zb.cpu().numpy())


def test_switching_host_buffers_fall_back_to_the_loop():
    hop, S, n, period = 256, 2, 40, 16
    ir0, x, dirs = _case(hop, S, 2048, n, period)
    a = T.TvolapEngine(T.partition(ir0, hop))
    b = T.TvolapEngine(T.partition(ir0, hop))
    ya = a.process_switching(x.cpu().numpy(), [None if d is None else d.cpu().numpy() for d in dirs], period)
    yb = _loop(b, x, dirs, period, hop)
    b.synchronize()  # device calls are asynchronous on the engine's stream
    assert np.array_equal(ya, yb.cpu().numpy())


def test_switching_matches_oracle():
    hop, S, taps, n, period = 256, 2, 2048, 50, 16
    ir0, x, dirs = _case(hop, S, taps, n, period)
    eng_g = T.TvolapEngine(T.partition(ir0, hop))
    y = eng_g.process_switching(x, dirs, period)
    eng_g.synchronize()
    y = y.cpu().numpy()
    xs = x.cpu().numpy().astype(np.float64)
    eng = O.Engine(O.partition(ir0.astype(np.float32).astype(np.float64), hop))
    ref = []
    for h in range(n):
        if h % period == 0 and dirs[h // period] is not None:
            eng.exchange_filter(O.partition(dirs[h // period].cpu().numpy().T.astype(np.float64), hop,
                                            eng.partition_count()))
        ref.append(eng.process(xs[:, h * hop:(h + 1) * hop].T))
    ref = np.concatenate(ref).T
    assert np.abs(y - ref).max() <= 1e-4 * np.abs(ref).max()


def test_switching_validation():
    import torch

    eng = T.TvolapEngine(T.partition(np.ones((100, 2)), 64))
    x = torch.zeros((2, 64 * 8), device="cuda")
    with pytest.raises(T.IncompatibleFilterError):
        eng.process_switching(x, [torch.zeros((3, 100), device="cuda")] * 8, 4)
    with pytest.raises(T.InvalidInputError):
        eng.process_switching(x, [None], 4)
    big = torch.zeros((2, 64 * 2 * 9), device="cuda")
    with pytest.raises(T.IncompatibleFilterError):
        eng.process_switching(x, [big] * 2, 4)


@pytest.mark.parametrize("n_hops,period,hop", [(16 * 9 + 5, 16, 256), (64, 16, 256), (90, 10, 256), (40, 8, 512),
                                              (50, 16, 256)])
def test_switching_pinned_host_pipeline(monkeypatch, n_hops, period, hop):
    """Pinned host buffers: chunked H2D / launch / D2H pipeline (switching kernel, or the loop on
    device staging for 2048-point transforms), bit-identical to the device call."""
    import torch

    T.set_default_tuning("wide", 0)  # device reference = the switching launch the pipeline runs
    S, taps = 4, 4096
    ir0, x, dirs = _case(hop, S, taps, n_hops, period, none_at=(1,))
    xh = x.cpu().pin_memory()
    irh = [None if d is None else d.cpu().pin_memory() for d in dirs]
    yh = torch.empty(xh.shape, dtype=torch.float32).pin_memory()
    a = T.TvolapEngine(T.partition(ir0, hop))
    b = T.TvolapEngine(T.partition(ir0, hop))
    a.process_switching(xh, irh, period, out=yh)
    a.synchronize()
    yd = b.process_switching(x, dirs, period)
    b.synchronize()
    assert np.array_equal(yh.numpy(), yd.cpu().numpy())
