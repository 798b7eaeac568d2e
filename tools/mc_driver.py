"""Monte-Carlo kernels once each at paper scale (for ncu): device draws + token counts,
4,096 trials of BalanceExperiment(LOCAL_PRESORT, snake, Topology(128, 8), lb 16), 10 M corpus."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2402_02447_b200 import BalanceExperiment, Topology  # noqa: E402
from paper_2402_02447_b200.mcsim import _prepare, draw_trials_device, trial_token_counts  # noqa: E402
from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths  # noqa: E402

lens = generate_lengths(LengthDistribution(), 10_000_000, 2402)
exp = BalanceExperiment("local_presort", Topology(128, 8), lens, seed=2402, local_batch=16, trials=4096, scan="snake")
prep = _prepare(exp)
for _ in range(2):
    mat = draw_trials_device(exp, 0, 4096, prep=prep)
    trial_token_counts(exp, mat, prep.max_len)
torch.cuda.synchronize()
print("mc_driver done")
