"""Repro: C5-geometry bank engine, single-hop process() calls with per-hop select_bank."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2310_00319_b200 import tvolap as T  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L, M, NB = 32, 512, 16
g = np.random.default_rng(0)
bank = g.standard_normal((NB, 1, 2 * L * M)).astype(np.float32) * 0.01
eng = T.TvolapBankEngine(bank, L, S)
print("geometry", eng.launch_config(), eng.block_config(), flush=True)
for h in range(4):
    eng.select_bank(g.integers(0, NB, S).astype(np.int32))
    y = eng.process(g.uniform(-1, 1, (L, S)))
    print(h, float(np.abs(y).max()), flush=True)
