"""TEST INFRASTRUCTURE: run a BASELINE config through the fp64 oracle on the same seeded inputs."""
from __future__ import annotations

from typing import Optional, Sequence

import numpy as np

import oracle as O
from paper_2310_00319_b200 import workload as W


def oracle_config(cfg: W.Config, n_hops: int, lane0: int = 0, sources: Optional[int] = None,
                  subset: Optional[Sequence[int]] = None, threads: Optional[int] = None,
                  which: Optional[str] = None):
    """Oracle outputs (len(subset)*ears, n_hops*L) for sources lane0+subset[i]; fp32-rounded inputs/IRs.

    which="ref" runs the reference's own engine (oracle/_ref, see oracle/oracle.py), "port" the
    restatement; default: the reference itself when its library is present (tests/test_ref_pin.py
    proves the two bit-identical)."""
    with O.using(which or best_oracle()):
        return _oracle_config(cfg, n_hops, lane0, sources, subset, threads)


def best_oracle() -> str:
    """"ref" (the reference's own sources, oracle/_ref) when built, else "port"."""
    return "ref" if O.ref_available() else "port"


def _oracle_config(cfg, n_hops, lane0, sources, subset, threads):
    sources = cfg.sources if sources is None else sources
    subset = list(range(sources)) if subset is None else list(subset)
    L = cfg.hop
    x = np.stack([W.white(cfg, lane0 + s, 1, 0, n_hops * L, dtype=np.float64)[0] for s in subset])
    threads = threads or W.host_threads()
    if cfg.mode == "bank":
        bank = W.bank_irs(cfg, dtype=np.float64)
        sched = W.schedule(cfg, 0, n_hops, lane0, sources)[:, subset]
        _, y = O.run_workload(L, cfg.partitions, len(subset), cfg.ears, n_hops, x, 1, bank_ir=bank,
                              schedule=np.ascontiguousarray(sched), threads=threads)
    else:
        n_sw = -(-n_hops // cfg.period)
        irs = np.stack([
            W.ir_items(cfg, [(lane0 + s, e, k) for s in subset for e in range(cfg.ears)], dtype=np.float64)
            .reshape(len(subset), cfg.ears, cfg.ir_length) for k in range(n_sw)])
        _, y = O.run_workload(L, cfg.partitions, len(subset), cfg.ears, n_hops, x, 0, fresh_ir=irs,
                              period=cfg.period, threads=threads)
    return y


def rel_err(got, ref) -> float:
    """max|got - ref| / max|ref| — the north-star parity metric."""
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-300))


TOL = 1e-4  # BASELINE.json north_star: max|y_gpu - y_ref| <= 1e-4 * max|y_ref| (fp32)
