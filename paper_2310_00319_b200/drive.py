"""Workload driver: streams a BASELINE config through the B200 engine.

The GPU-side counterpart of the reference's drive() loop
(proj/src/experiment.cpp:33-54): a filter change is staged right before the hop
it applies to (experiment.cpp:44-45, test_engine.cpp:127-131), hops are fed in
order, outputs come back per lane. Fresh-IR configs (C2, C4) use
exchange_filter with a newly generated IR set every `period` hops; bank configs
(C1, C3, C5) pass a per-hop bank schedule to process_hops.
"""
from __future__ import annotations

from typing import Optional

import numpy as np

from . import workload as W
from .tvolap import TvolapBankEngine, TvolapEngine, partition


def make_engine(cfg: W.Config, lane0: int = 0, sources: Optional[int] = None, device: int = 0):
    sources = cfg.sources if sources is None else sources
    if cfg.mode == "bank":
        eng = TvolapBankEngine(W.bank_irs(cfg), cfg.hop, sources, min_partitions=cfg.partitions, device=device)
    else:
        ir0 = W.fresh_irs(cfg, 0, lane0, sources)[:, 0, :]  # (sources, taps)
        eng = TvolapEngine(partition(ir0.T, cfg.hop, cfg.partitions), device=device)
    return eng


def run_host(cfg: W.Config, n_hops: int, lane0: int = 0, sources: Optional[int] = None, device: int = 0,
             x: Optional[np.ndarray] = None, engine=None):
    """Run n_hops of cfg from zero state with host numpy buffers. Returns (engine, out (lanes, n_hops*L))."""
    sources = cfg.sources if sources is None else sources
    L = cfg.hop
    if x is None:
        x = W.white(cfg, lane0, sources, 0, n_hops * L)
    eng = engine or make_engine(cfg, lane0, sources, device)
    out = np.empty((sources * cfg.ears, n_hops * L), dtype=np.float32)
    if cfg.mode == "bank":
        sched = W.schedule(cfg, 0, n_hops, lane0, sources)
        eng.process_hops(x, out=out, schedule=sched)
    else:
        for h0 in range(0, n_hops, cfg.period):
            k = h0 // cfg.period
            if k:
                irk = W.fresh_irs(cfg, k, lane0, sources)[:, 0, :]
                eng.exchange_filter(partition(irk.T, L, cfg.partitions))
            h1 = min(n_hops, h0 + cfg.period)
            eng.process_hops(np.ascontiguousarray(x[:, h0 * L:h1 * L]), out=out[:, h0 * L:h1 * L])
    return eng, out
