"""Monte-Carlo balance engine on the GPU vs the reference.

Golden per-trial token counts, BalanceStats and an ablation table come from
running ddpsim.mcsim itself (tests/golden/h2_mc_golden.json); the paper-scale
case (1,024 GPUs, 10 M corpus) is checked trial by trial against the oracle.
Integer work: everything is ``==``, including the float statistics (the
aggregation is the reference's own numpy expression on exact int64 arrays).
"""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import ddp_oracle as O
from paper_2402_02447_b200 import Topology
from paper_2402_02447_b200.mcsim import (BalanceExperiment, _prepare, draw_trials, run_ablation,
                                         run_balance_experiment, trial_token_counts)

pytestmark = pytest.mark.gpu
GOLDEN = json.loads((Path(__file__).parent / "golden" / "h2_mc_golden.json").read_text())


def _exp(c, lengths, **kw):
    return BalanceExperiment(c["strategy"], Topology(c["nodes"], c["gpn"]), lengths, seed=c["seed"],
                             local_batch=c["lb"], trials=c["trials"], scan=c["scan"], **kw)


@pytest.mark.parametrize("case", range(len(GOLDEN["cases"])))
def test_mc_engine_matches_reference_trials_and_stats(case):
    c = GOLDEN["cases"][case]
    lengths = O.generate_lengths(GOLDEN["corpus_n"], GOLDEN["corpus_seed"])
    exp = _exp(c, lengths)
    prep = _prepare(exp)
    mat = torch.from_numpy(draw_trials(exp, 0, c["trials"], prep=prep)).cuda()
    mins, maxs, cnt, bad = trial_token_counts(exp, mat, prep.max_len, counts=True)
    assert int(bad) == 0
    assert cnt.cpu().tolist() == c["tokens"]
    assert mins.cpu().tolist() == [min(t) for t in c["tokens"]]
    assert maxs.cpu().tolist() == [max(t) for t in c["tokens"]]
    st = run_balance_experiment(exp, chunk=7)  # several chunks: the double-buffered pipeline
    assert st.__dict__ == c["stats"]


def test_mc_ablation_matches_reference():
    a = GOLDEN["ablation"]
    lengths = O.generate_lengths(GOLDEN["corpus_n"], GOLDEN["corpus_seed"])
    base = BalanceExperiment("local_presort", Topology(a["nodes"], a["gpn"]), lengths, seed=a["seed"],
                             local_batch=a["lb"], trials=a["trials"])
    rows = run_ablation(base)
    assert [[label, st.__dict__] for label, st in rows] == a["rows"]


@pytest.mark.parametrize("strategy,scan", [("local_presort", "snake"), ("global_presort", "raster"),
                                           ("stratified", "raster")])
def test_mc_engine_paper_scale_vs_oracle(strategy, scan):
    """1,024 GPUs (128 nodes x 8), lb 16, the 10 M corpus: 64 trials on the GPU,
    trials 0, 31 and 63 recomputed by the oracle."""
    lengths = O.generate_lengths(10_000_000, 2402)
    exp = BalanceExperiment(strategy, Topology(128, 8), lengths, seed=99, local_batch=16, trials=64, scan=scan)
    prep = _prepare(exp)
    mat = torch.from_numpy(draw_trials(exp, 0, 64, prep=prep)).cuda()
    mins, maxs, cnt, bad = trial_token_counts(exp, mat, prep.max_len, counts=True)
    assert int(bad) == 0
    cnt = cnt.cpu().numpy()
    for t in (0, 31, 63):
        ref = O.mcsim_trial_counts(strategy, lengths, O.DEFAULT_BOUNDS, 16, 128, 8, scan == "snake", 99, t)
        assert cnt[t].tolist() == ref.tolist(), t
    assert np.array_equal(mins.cpu().numpy(), cnt.min(axis=1))
    assert np.array_equal(maxs.cpu().numpy(), cnt.max(axis=1))


@pytest.mark.parametrize("case", range(len(GOLDEN["cases"])))
def test_device_draws_equal_host_draws(case):
    """b2_mc_draw_device (one warp per trial) == b2_mc_draw (host threads) == numpy, bit for bit."""
    from paper_2402_02447_b200.mcsim import draw_trials_device

    c = GOLDEN["cases"][case]
    lengths = O.generate_lengths(GOLDEN["corpus_n"], GOLDEN["corpus_seed"])
    exp = _exp(c, lengths)
    prep = _prepare(exp)
    host = draw_trials(exp, 5, 30, prep=prep)
    dev = draw_trials_device(exp, 5, 30, prep=prep)
    assert dev is not None
    assert np.array_equal(dev.cpu().numpy(), host)


@pytest.mark.parametrize("pmax", ["1", "3"])
def test_device_draws_compact_set_redo_path(pmax, monkeypatch):
    """The compact (16-bit entry) Floyd set marks a trial whose probe index overflows and the
    32-bit kernel redoes it: with the probe cap forced down most trials take that path, some
    don't -- every trial still equals the host draws bit for bit."""
    from paper_2402_02447_b200.mcsim import draw_trials_device

    lengths = O.generate_lengths(10_000_000, 2402)
    exp = BalanceExperiment("local_presort", Topology(128, 8), lengths, seed=9, local_batch=16, trials=48)
    prep = _prepare(exp)
    want = draw_trials(exp, 3, 48, prep=prep)
    monkeypatch.setenv("B2_MC_DRAW16_PMAX", pmax)
    dev = draw_trials_device(exp, 3, 48, prep=prep)
    assert np.array_equal(dev.cpu().numpy(), want)


def test_device_draws_paper_scale_and_tail_shuffle_fallback():
    from paper_2402_02447_b200.mcsim import draw_trials_device, run_trials

    lengths = O.generate_lengths(10_000_000, 2402)
    for strategy in ("local_presort", "none"):
        exp = BalanceExperiment(strategy, Topology(128, 8), lengths, seed=4, local_batch=16, trials=40)
        prep = _prepare(exp)
        dev = draw_trials_device(exp, 0, 40, prep=prep)
        assert np.array_equal(dev.cpu().numpy(), draw_trials(exp, 0, 40, prep=prep))
    # 20,000-sample corpus, 32 GPUs x lb 16 = 512 > 20,000 // 50: numpy's tail-shuffle branch
    small = O.generate_lengths(20_000, 606)
    exp = BalanceExperiment("none", Topology(4, 8), small, seed=8, local_batch=16, trials=25)
    assert draw_trials_device(exp, 0, 25) is None
    mins, maxs = run_trials(exp)  # auto: falls back to host draws
    ref = [O.mcsim_trial_counts("none", small, O.DEFAULT_BOUNDS, 16, 4, 8, False, 8, t) for t in range(25)]
    assert mins.tolist() == [int(r.min()) for r in ref] and maxs.tolist() == [int(r.max()) for r in ref]
