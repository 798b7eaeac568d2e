"""Generate golden fixtures by running the REFERENCE (ddpsim 0.1.0) itself.

Run in the build container only (needs /root/reference, read-only):

    python tests/golden/make_golden.py

Writes ``tests/golden/h1_golden.npz``, ``h2_golden.json`` and ``h2_mc_golden.json``.
These pin the oracle (``oracle/ddp_oracle.py``) and, through it, the CUDA
path.  Nothing on the GPU box reads /root/reference; the fixtures travel with
the repo.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from ddpsim import balance, gradsync, mcsim, seqdata, strata  # noqa: E402

OUT = Path(__file__).resolve().parent


def h1_cases():
    rng = np.random.default_rng(24020)
    cases = {}
    # (K, D, B, scale) — mixes clipped / unclipped buckets, uneven last bucket
    specs = [
        (1, 8, 4, 1.0), (1, 7, 3, 10.0), (2, 7, 3, 10.0), (4, 10, 1, 3.0),
        (1, 4096, 4, 0.01), (1, 4099, 5, 0.05), (3, 3001, 7, 0.02), (8, 2048, 4, 1.0),
        (16, 600, 25, 0.3), (5, 12, 4, 0.005), (1, 65537, 3, 0.004), (4, 1000, 1, 30.0),
    ]
    for i, (k, d, b, scale) in enumerate(specs):
        # fp32-representable inputs so the fp32 device path sees the same values
        w = (rng.normal(size=(k, d)) * scale).astype(np.float32).astype(np.float64)
        layout = gradsync.equal_bucket_layout(d, b)
        st = gradsync.GradientState(w.copy(), layout)
        out = gradsync.sync_bucketwise(st, gradsync.ClipConfig(1.0, "bucket_wise"))
        norms = np.array([[np.linalg.norm(w[kk, a:z]) for a, z in layout] for kk in range(k)])
        cases[f"c{i}_workers"] = w
        cases[f"c{i}_layout"] = np.array(layout, dtype=np.int64)
        cases[f"c{i}_out"] = out
        cases[f"c{i}_norms"] = norms
        if b == 1:
            cases[f"c{i}_before"] = gradsync.sync_before(
                gradsync.GradientState(w.copy(), layout), gradsync.ClipConfig(1.0, "before_allreduce")
            )
            cases[f"c{i}_after"] = gradsync.sync_after(
                gradsync.GradientState(w.copy(), layout), gradsync.ClipConfig(1.0, "after_allreduce")
            )
    # clip_by_norm KATs incl. the inclusive edge
    kat_in = [np.array([3.0, 4.0]), np.array([0.0, 2.0]), np.zeros(4), np.array([3.0, 4.0])]
    kat_lim = [1.0, 2.0, 0.5, 10.0]
    for j, (g, lim) in enumerate(zip(kat_in, kat_lim)):
        cases[f"kat{j}_in"] = g
        cases[f"kat{j}_limit"] = np.array(lim)
        cases[f"kat{j}_out"] = gradsync.clip_by_norm(g, lim)
    cases["n_cases"] = np.array(len(specs))
    cases["n_kats"] = np.array(len(kat_in))
    np.savez_compressed(OUT / "h1_golden.npz", **cases)


def h2_cases():
    doc: dict = {}
    # generate_corpus + stratify at a few seeds / sizes
    corp = []
    for n, seed in ((5000, 2402), (777, 7), (20000, 55)):
        samples = seqdata.generate_corpus(seqdata.LengthDistribution(), n, seed)
        st = strata.stratify(samples, strata.DEFAULT_STRATUM_BOUNDARIES)
        corp.append({
            "n": n, "seed": seed,
            "lengths": [s.length for s in samples],
            "pools": [[s.id for s in pool] for pool in st.buckets],
            "probs": list(st.probs),
            "alloc16": list(strata.allocate_counts(st.probs, 16).counts),
            "alloc48": list(strata.allocate_counts(st.probs, 48).counts),
        })
    doc["corpora"] = corp
    # custom boundaries with boundary-equal lengths
    samples = [seqdata.Sample(i, x) for i, x in enumerate([128, 129, 256, 257, 1, 512, 384, 385, 64])]
    st = strata.stratify(samples, (128, 256, 384, 512))
    doc["edge_stratify"] = {
        "lengths": [s.length for s in samples],
        "pools": [[s.id for s in p] for p in st.buckets],
        "probs": list(st.probs),
    }
    # allocate_counts table
    alloc = []
    rng = np.random.default_rng(99)
    for _ in range(40):
        k = int(rng.integers(1, 8))
        p = rng.random(k)
        p[rng.random(k) < 0.2] = 0.0
        if p.sum() == 0:
            p[0] = 1.0
        lb = int(rng.integers(0, 200))
        alloc.append({"probs": p.tolist(), "lb": lb, "counts": list(strata.allocate_counts(p, lb).counts)})
    doc["allocate"] = alloc
    # draw_batch epoch walks (pins the RNG draw order + swap-pop + borrowing)
    draws = []
    for n, seed, lb, bounds in ((3000, 11, 16, (128, 256, 384, 512)), (500, 12, 48, (128, 256, 384, 512)),
                                (256, 13, 10, (100, 300, 512))):
        samples = seqdata.generate_corpus(seqdata.LengthDistribution(), n, seed)
        st = strata.stratify(samples, bounds)
        al = strata.allocate_counts(st.probs, lb)
        seq = []
        step = 0
        while True:
            try:
                batch = strata.draw_batch(st, al, seed=1000 + step)
            except ValueError as e:
                seq.append({"error": str(e)})
                break
            seq.append([s.id for s in batch])
            step += 1
            if step >= 60:
                break
        draws.append({"n": n, "seed": seed, "lb": lb, "bounds": list(bounds),
                      "counts": list(al.counts), "batches": seq})
    doc["draws"] = draws
    # local presort over real draws (2 nodes x 4 GPUs, lb 16/48; both scans)
    lp = []
    for nodes, gpn, lb, seed in ((1, 8, 16, 21), (2, 4, 48, 22), (1, 4, 12, 23), (4, 2, 6, 24)):
        samples = seqdata.generate_corpus(seqdata.LengthDistribution(), 20000, seed)
        by_id = {s.id: s for s in samples}
        topo = seqdata.Topology(nodes, gpn)
        for step in range(3):
            per_gpu = []
            for g in range(topo.total_gpus):
                shard = samples[g::topo.total_gpus]
                st = strata.stratify(shard)
                al = strata.allocate_counts(st.probs, lb)
                per_gpu.append(strata.draw_batch(st, al, seed=seed * 100 + step * 10 + g))
            for scan in ("snake", "raster"):
                a = balance.assign_local_presort(per_gpu, topo, scan)
                lp.append({
                    "nodes": nodes, "gpn": gpn, "scan": scan,
                    "draw_ids": [[s.id for s in d] for d in per_gpu],
                    "draw_lens": [[by_id[s.id].length for s in d] for d in per_gpu],
                    **a.to_dict(),
                })
    # ties: duplicate lengths so the id tie-break decides
    rng = np.random.default_rng(5)
    for scan in ("snake", "raster"):
        ids = rng.permutation(64)
        lens = rng.integers(1, 4, size=64)
        samples = [seqdata.Sample(int(i), int(x)) for i, x in zip(ids, lens)]
        per_gpu = [samples[g * 16:(g + 1) * 16] for g in range(4)]
        a = balance.assign_local_presort(per_gpu, seqdata.Topology(1, 4), scan)
        lp.append({"nodes": 1, "gpn": 4, "scan": scan,
                   "draw_ids": [[s.id for s in d] for d in per_gpu],
                   "draw_lens": [[s.length for s in d] for d in per_gpu], **a.to_dict()})
    doc["local_presort"] = lp
    # global presort (whole batch is one segment)
    gp = []
    for scan in ("raster", "snake"):
        samples = seqdata.generate_corpus(seqdata.LengthDistribution(), 96, 31)
        a = balance.assign_global_presort(samples, seqdata.Topology(2, 4), scan)
        gp.append({"scan": scan, "gpus": 8, "ids": [s.id for s in samples],
                   "lens": [s.length for s in samples], **a.to_dict()})
    doc["global_presort"] = gp
    # mcsim LOCAL_PRESORT trial: capture the (b, G) matrix and the token counts
    mc = []
    corpus = tuple(seqdata.generate_corpus(seqdata.LengthDistribution(), 50_000, 505))
    for nodes, gpn, lb, scan in ((1, 8, 16, "snake"), (2, 4, 48, "raster"), (8, 8, 16, "snake")):
        exp = mcsim.BalanceExperiment("local_presort", seqdata.Topology(nodes, gpn), corpus,
                                      seed=55, local_batch=lb, trials=3, scan=scan)
        prep = mcsim._prepare(exp)
        for t in range(3):
            from ddpsim.seeding import derive_rng
            mat = mcsim._stratified_matrix(derive_rng(55, t), prep, nodes * gpn)
            tok = mcsim._trial_token_counts(derive_rng(55, t), exp, prep)
            mc.append({"nodes": nodes, "gpn": gpn, "scan": scan, "mat": mat.tolist(),
                       "tokens": tok.tolist()})
    doc["mcsim"] = mc
    (OUT / "h2_golden.json").write_text(json.dumps(doc, separators=(",", ":")))


def mc_cases():
    """mcsim: per-trial token counts of every strategy the
    GPU engine covers, plus the aggregated BalanceStats and one ablation table,
    all computed by the reference itself."""
    from ddpsim import mcsim, seqdata
    from ddpsim.seeding import derive_rng

    n, cseed = 20_000, 606
    corpus = tuple(seqdata.generate_corpus(seqdata.LengthDistribution(), n, cseed))
    cases = []
    for strat, scan, nodes, gpn, lb in (("none", "raster", 2, 4, 16), ("stratified", "raster", 1, 8, 16),
                                        ("local_presort", "raster", 2, 4, 16), ("local_presort", "snake", 4, 8, 16),
                                        ("local_presort", "snake", 1, 8, 48), ("global_presort", "raster", 2, 4, 16),
                                        ("global_presort", "snake", 4, 8, 8)):
        exp = mcsim.BalanceExperiment(strat, seqdata.Topology(nodes, gpn), corpus, seed=77, local_batch=lb,
                                      trials=40, scan=scan)
        prep = mcsim._prepare(exp)
        tokens = [mcsim._trial_token_counts(derive_rng(77, t), exp, prep).tolist() for t in range(exp.trials)]
        st = mcsim.run_balance_experiment(exp)
        cases.append({"strategy": strat, "scan": scan, "nodes": nodes, "gpn": gpn, "lb": lb, "seed": 77,
                      "trials": exp.trials, "tokens": tokens, "stats": st.__dict__})
    base = mcsim.BalanceExperiment("local_presort", seqdata.Topology(2, 4), corpus, seed=2402, local_batch=16,
                                   trials=25)
    ablation = [[label, st.__dict__] for label, st in mcsim.run_ablation(base)]
    doc = {"corpus_n": n, "corpus_seed": cseed, "cases": cases,
           "ablation": {"nodes": 2, "gpn": 4, "lb": 16, "seed": 2402, "trials": 25, "rows": ablation}}
    (OUT / "h2_mc_golden.json").write_text(json.dumps(doc, separators=(",", ":")))


def timeline_cases():
    """timeline.schedule totals (timeline.py:97-152) for seeded random plans:
    pins the restated model in tools/timeline_calibrate.py."""
    from ddpsim import timeline

    rng = np.random.default_rng(8)
    cases = []
    for B in (1, 2, 5, 37, 52):
        for scale in (0.1, 1.0, 10.0):
            plan = timeline.TimelinePlan(t_comp=tuple(rng.uniform(0.5, 3, B)), t_comm=tuple(rng.uniform(0, 1, B) * scale),
                                         t_clip=tuple(rng.uniform(0, 0.1, B)), t_gclip=float(rng.uniform(0, 2)),
                                         t_nred=float(rng.uniform(0, 0.5)))
            cases.append({"t_comp": list(plan.t_comp), "t_comm": list(plan.t_comm), "t_clip": list(plan.t_clip),
                          "t_gclip": plan.t_gclip, "t_nred": plan.t_nred,
                          "total": {m: timeline.schedule(plan, m).total
                                    for m in ("bucket_wise", "after_allreduce", "before_allreduce")}})
    (OUT / "timeline_golden.json").write_text(json.dumps(cases))


if __name__ == "__main__":
    h1_cases()
    h2_cases()
    mc_cases()
    timeline_cases()
    for f in sorted(OUT.glob("h*_golden.*")):
        print(f.name, f.stat().st_size)
