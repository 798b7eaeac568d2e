"""Pin the CPU oracle against the reference's golden vectors and KATs (no GPU).

The fixtures under tests/golden/ were produced by running the reference
(ddpsim 0.1.0) itself — see tests/golden/make_golden.py.
"""

import numpy as np
import pytest

from oracle import ddp_oracle as O


# ---------------------------------------------------------------- H1
def test_h1_sync_bucketwise_matches_reference(h1_golden):
    g = h1_golden
    for i in range(int(g["n_cases"])):
        w = g[f"c{i}_workers"]
        layout = [tuple(x) for x in g[f"c{i}_layout"]]
        out = O.sync_bucketwise(w, layout, 1.0)
        # same numpy ops in the same order -> bit-identical
        assert out.tobytes() == g[f"c{i}_out"].tobytes(), i
        norms = np.array([O.bucket_norms(w[k], layout) for k in range(w.shape[0])])
        assert norms.tobytes() == g[f"c{i}_norms"].tobytes()
        if f"c{i}_before" in g:
            np.testing.assert_array_equal(O.sync_before(w, 1.0), g[f"c{i}_before"])
            np.testing.assert_array_equal(O.sync_after(w, 1.0), g[f"c{i}_after"])


def test_h1_clip_kats(h1_golden):
    g = h1_golden
    for j in range(int(g["n_kats"])):
        out = O.clip_by_norm(g[f"kat{j}_in"], float(g[f"kat{j}_limit"]))
        np.testing.assert_array_equal(out, g[f"kat{j}_out"])
    # test_gradsync.py:31-44
    np.testing.assert_allclose(O.clip_by_norm(np.array([3.0, 4.0]), 1.0), [0.6, 0.8], atol=1e-15)
    np.testing.assert_array_equal(O.clip_by_norm(np.array([0.0, 2.0]), 2.0), [0.0, 2.0])
    with pytest.raises(ValueError, match="non-finite"):
        O.clip_by_norm(np.array([1.0, np.inf]), 1.0)


def test_h1_layout_kats():
    # test_gradsync.py:147-151, 218-220
    assert O.equal_bucket_layout(7, 3) == ((0, 2), (2, 4), (4, 7))
    assert O.equal_bucket_layout(10, 3) == ((0, 3), (3, 6), (6, 10))
    assert O.equal_bucket_layout(4, 4) == ((0, 1), (1, 2), (2, 3), (3, 4))
    with pytest.raises(ValueError):
        O.equal_bucket_layout(3, 4)


def test_h1_hand_bucket_kat():
    # test_gradsync.py:135-141
    out = O.sync_bucketwise(np.array([[3.0, 4.0] * 4]), O.equal_bucket_layout(8, 4), 1.0)
    np.testing.assert_allclose(out, [0.3, 0.4] * 4, atol=1e-15)


def test_h1_allreduce_pairwise_tree():
    np.testing.assert_array_equal(O.allreduce_mean([[1.0, 2.0], [3.0, 4.0]]), [2.0, 3.0])
    rng = np.random.default_rng(0)
    for k in (1, 2, 3, 5, 8, 16):
        w = rng.normal(size=(k, 33))
        np.testing.assert_allclose(O.allreduce_mean(w), w.mean(axis=0), rtol=1e-12, atol=1e-15)


# ---------------------------------------------------------------- H2
def test_h2_generate_and_stratify(h2_golden):
    for c in h2_golden["corpora"]:
        lens = O.generate_lengths(c["n"], c["seed"])
        assert lens.tolist() == c["lengths"]
        pools, probs = O.stratify(lens)
        assert [p.tolist() for p in pools] == c["pools"]
        assert list(probs) == c["probs"]
        assert list(O.allocate_counts(probs, 16)) == c["alloc16"]
        assert list(O.allocate_counts(probs, 48)) == c["alloc48"]
    e = h2_golden["edge_stratify"]
    pools, probs = O.stratify(e["lengths"])
    assert [p.tolist() for p in pools] == e["pools"]
    assert list(probs) == e["probs"]


def test_h2_stratify_kats():
    # test_strata.py:19-47
    pools, probs = O.stratify([100, 200, 300, 500])
    assert [len(p) for p in pools] == [1, 1, 1, 1] and probs == (0.25,) * 4
    pools, _ = O.stratify([128, 129, 256, 257])
    assert [len(p) for p in pools] == [1, 2, 1, 0]
    pools, _ = O.stratify([10, 300, 20, 5, 290])
    assert pools[0].tolist() == [0, 2, 3] and pools[2].tolist() == [1, 4]
    with pytest.raises(ValueError, match="id 7"):
        O.stratify([100, 600], ids=[0, 7])
    with pytest.raises(ValueError):
        O.stratify([])


def test_h2_allocate(h2_golden):
    for a in h2_golden["allocate"]:
        assert list(O.allocate_counts(a["probs"], a["lb"])) == a["counts"]
    assert O.allocate_counts((5 / 16, 2 / 16, 3 / 16, 6 / 16), 16) == (5, 2, 3, 6)
    assert O.allocate_counts((0.373, 0.197, 0.117, 0.314), 16) == (6, 3, 2, 5)
    assert O.allocate_counts((0.5, 0.5), 3) == (2, 1)


def test_h2_draw_batch_epochs(h2_golden):
    for d in h2_golden["draws"]:
        lens = O.generate_lengths(d["n"], d["seed"])
        pools, probs = O.stratify(lens, d["bounds"])
        pools = [p.tolist() for p in pools]
        counts = O.allocate_counts(probs, d["lb"])
        assert list(counts) == d["counts"]
        for step, expect in enumerate(d["batches"]):
            if isinstance(expect, dict):
                with pytest.raises(ValueError) as ei:
                    O.draw_batch(pools, d["bounds"], counts, seed=1000 + step)
                assert str(ei.value) == expect["error"]
            else:
                assert O.draw_batch(pools, d["bounds"], counts, seed=1000 + step) == expect


def test_h2_local_presort(h2_golden):
    for c in h2_golden["local_presort"]:
        per_gpu, tok = O.assign_local_presort(
            c["draw_ids"], c["draw_lens"], c["nodes"], c["gpn"], c["scan"] == "snake"
        )
        assert per_gpu == c["per_gpu_ids"]
        assert list(tok) == c["token_counts"]


def test_h2_local_presort_kats():
    # test_balance.py:138-146
    lens = list(range(16, 0, -1))
    ids = list(range(16))
    dl = [lens[g * 4:(g + 1) * 4] for g in range(4)]
    di = [ids[g * 4:(g + 1) * 4] for g in range(4)]
    assert O.assign_local_presort(di, dl, 1, 4, True)[1] == (34, 34, 34, 34)
    assert O.assign_local_presort(di, dl, 1, 4, False)[1] == (40, 36, 32, 28)
    with pytest.raises(ValueError, match="differ"):
        O.assign_local_presort([[0, 1], [2]], [[1, 2], [3]], 1, 2)


def test_h2_global_presort(h2_golden):
    for c in h2_golden["global_presort"]:
        out, tok = O.presort_deal_segments(c["ids"], c["lens"], len(c["ids"]), c["gpus"],
                                           c["scan"] == "snake")
        assert out[0].tolist() == c["per_gpu_ids"]
        assert tok[0].tolist() == c["token_counts"]


def test_h2_mcsim_second_oracle(h2_golden):
    for c in h2_golden["mcsim"]:
        tok = O.mcsim_local_presort_tokens(c["mat"], c["nodes"], c["gpn"], c["scan"] == "snake")
        assert tok.tolist() == c["tokens"]


# ---------------------------------------------------------------------------
# mcsim: the oracle vs the reference's own trials

def _mc_golden():
    import json
    from pathlib import Path

    return json.loads((Path(__file__).parent / "golden" / "h2_mc_golden.json").read_text())


def test_oracle_mcsim_trials_and_stats_match_reference():
    g = _mc_golden()
    lengths = O.generate_lengths(g["corpus_n"], g["corpus_seed"])
    for c in g["cases"]:
        mins, maxs = [], []
        for t in range(c["trials"]):
            tok = O.mcsim_trial_counts(c["strategy"], lengths, O.DEFAULT_BOUNDS, c["lb"], c["nodes"], c["gpn"],
                                       c["scan"] == "snake", c["seed"], t)
            assert tok.tolist() == c["tokens"][t], (c["strategy"], c["scan"], t)
            mins.append(tok.min())
            maxs.append(tok.max())
        assert O.mcsim_stats(mins, maxs) == c["stats"], c["strategy"]
