"""H1 parity on the GPU: CUDA path vs the reference golden vectors and the oracle.

Tolerances (north_star): norms and clipped gradients within 1e-5 relative in
fp32 (max |diff| <= 1e-5 * max |ref|); the fp64 device path is held to 1e-12;
a bf16 comm buffer is held to bf16 rounding (2^-8 relative per element).
"""

import math

import numpy as np
import pytest
import torch

from oracle import ddp_oracle as O

pytestmark = pytest.mark.gpu

from paper_2402_02447_b200 import (  # noqa: E402
    BucketClipper,
    ClipConfig,
    GradientState,
    allreduce_mean,
    clip_by_norm,
    equal_bucket_layout,
    sync_after,
    sync_before,
    sync_bucketwise,
    synchronize,
)
from paper_2402_02447_b200 import synthetic  # noqa: E402

BUCKET = ClipConfig(1.0, "bucket_wise")
BEFORE = ClipConfig(1.0, "before_allreduce")
AFTER = ClipConfig(1.0, "after_allreduce")
F32_REL = 1e-5
F64_REL = 1e-12


def rel_err(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(np.abs(b).max(), 1e-300)
    return float(np.abs(a - b).max() / scale)


def state(workers, buckets=1):
    w = np.asarray(workers, dtype=float)
    return GradientState(w, equal_bucket_layout(w.shape[1], buckets))


# ------------------------------------------------------------- golden vectors
def test_golden_fp64_path(h1_golden):
    g = h1_golden
    for i in range(int(g["n_cases"])):
        w = g[f"c{i}_workers"]
        layout = [tuple(x) for x in g[f"c{i}_layout"]]
        out = sync_bucketwise(GradientState(w, layout), BUCKET)
        assert isinstance(out, np.ndarray) and out.dtype == np.float64
        # fp64 device path: 1e-12 of the vector's scale (norms differ from OpenBLAS ddot in the last bits)
        assert rel_err(out, g[f"c{i}_out"]) <= F64_REL, i
        if f"c{i}_before" in g:
            assert rel_err(sync_before(GradientState(w, layout), BEFORE), g[f"c{i}_before"]) <= F64_REL
            assert rel_err(sync_after(GradientState(w, layout), AFTER), g[f"c{i}_after"]) <= F64_REL


def test_golden_fp32_device_path(h1_golden):
    g = h1_golden
    for i in range(int(g["n_cases"])):
        w = g[f"c{i}_workers"]  # fp32-representable values
        layout = [tuple(x) for x in g[f"c{i}_layout"]]
        wt = torch.tensor(w, dtype=torch.float32, device="cuda")
        out = sync_bucketwise(GradientState(wt, layout), BUCKET)
        assert out.is_cuda and out.dtype == torch.float32
        assert rel_err(out.cpu().numpy(), g[f"c{i}_out"]) <= F32_REL, i


def test_golden_norms(h1_golden):
    g = h1_golden
    c = BucketClipper()
    for i in range(int(g["n_cases"])):
        w = g[f"c{i}_workers"]
        layout = [tuple(x) for x in g[f"c{i}_layout"]]
        K = w.shape[0]
        # fp64 input: exact fp64 accumulation; fp32 input: fp32 mini-sums of <= 8
        # squares promoted to fp64 (rel. error well below the 1e-5 contract)
        for dt, tol in ((torch.float64, 1e-13), (torch.float32, 1e-6)):
            wt = torch.tensor(w, dtype=dt, device="cuda")
            segs = [(k * w.shape[1] + a, 0, b - a) for k in range(K) for a, b in layout]
            norms = torch.empty(len(segs), dtype=torch.float64, device="cuda")
            c.clip_cast(wt, None, segs, 0.5, norms=norms)
            np.testing.assert_allclose(norms.cpu().numpy(), g[f"c{i}_norms"].ravel(), rtol=tol)


# ------------------------------------------------------------- reference KATs
def test_clip_kats():
    np.testing.assert_allclose(clip_by_norm(np.array([3.0, 4.0]), 1.0), [0.6, 0.8], atol=1e-15)
    g = np.array([3.0, 4.0])
    np.testing.assert_array_equal(clip_by_norm(g, 10.0), g)
    assert clip_by_norm(g, 10.0) is g  # not clipped: the same array object (gradsync.py:116)
    t = torch.tensor([3.0, 4.0], device="cuda")
    assert clip_by_norm(t, 10.0) is t
    np.testing.assert_array_equal(clip_by_norm(np.zeros(4), 0.5), np.zeros(4))
    # inclusive edge: norm == limit -> coefficient exactly 1 (test_gradsync.py:42-44)
    np.testing.assert_array_equal(clip_by_norm(np.array([0.0, 2.0]), 2.0), [0.0, 2.0])
    with pytest.raises(ValueError, match="non-finite"):
        clip_by_norm(np.array([1.0, np.inf]), 1.0)
    with pytest.raises(ValueError, match="non-finite"):
        clip_by_norm(np.array([np.nan]), 1.0)
    with pytest.raises(ValueError):
        clip_by_norm(np.ones(2), 0.0)
    # fp32 device tensor flavour of the inclusive edge
    t = torch.tensor([0.0, 2.0], device="cuda")
    assert torch.equal(clip_by_norm(t, 2.0), t)


def test_allreduce_kats():
    np.testing.assert_array_equal(allreduce_mean([[1.0, 2.0], [3.0, 4.0]]), [2.0, 3.0])
    np.testing.assert_array_equal(allreduce_mean([[5.0, -1.0]]), [5.0, -1.0])
    v = [1.5, 2.5, -3.0]
    np.testing.assert_array_equal(allreduce_mean([v, v, v]), v)
    with pytest.raises(ValueError, match="mismatch|matrix"):
        allreduce_mean([[1.0, 2.0], [3.0]])
    rng = np.random.default_rng(0)
    for k in (1, 2, 3, 5, 8, 16, 63, 64, 65, 100, 257):
        w = rng.normal(size=(k, 33))
        # the pairwise tree is the reference's: bit-identical to the oracle, for any K
        np.testing.assert_array_equal(allreduce_mean(w), O.allreduce_mean(w))
    w = rng.normal(size=(130, 1000))  # > 64 workers through sync_bucketwise (no K cap)
    # (clipped: the fp64 norm's summation order differs from BLAS ddot -> 1e-12, the fp64 bar)
    np.testing.assert_allclose(sync_bucketwise(state(w, 3), BUCKET),
                               O.sync_bucketwise(w, equal_bucket_layout(1000, 3), 1.0), rtol=1e-12, atol=1e-18)


def test_bucketwise_kats():
    out = sync_bucketwise(state([[3.0, 4.0] * 4], buckets=4), BUCKET)
    np.testing.assert_allclose(out, [0.3, 0.4] * 4, atol=1e-15)
    assert abs(np.linalg.norm(out) - 1.0) < 1e-12
    np.testing.assert_array_equal(sync_bucketwise(state(np.zeros((3, 12)), 4), BUCKET), np.zeros(12))
    st = GradientState(np.ones((2, 7)) * 10, equal_bucket_layout(7, 3))
    assert np.linalg.norm(sync_bucketwise(st, BUCKET)) <= 1.0 + 1e-9
    with pytest.raises(ValueError, match="mode"):
        sync_after(state([[1.0, 2.0]]), BEFORE)
    with pytest.raises(ValueError, match="non-finite"):
        GradientState(np.array([[1.0, np.nan]]), ((0, 2),))
    with pytest.raises(ValueError, match="non-finite"):
        GradientState(torch.tensor([[1.0, float("inf")]], device="cuda"), ((0, 2),))


def test_cross_mode_properties():
    rng = np.random.default_rng(7)
    for _ in range(60):
        k = int(rng.choice([1, 4, 16]))
        b = int(rng.choice([1, 4, 25]))
        d = int(rng.integers(b, 300))
        w = rng.normal(size=(k, d)) * float(rng.choice([0.01, 1.0, 100.0]))
        out = sync_bucketwise(state(w, b), BUCKET)
        assert np.linalg.norm(out) <= 1.0 + 1e-9
        assert rel_err(out, O.sync_bucketwise(w, equal_bucket_layout(d, b), 1.0)) <= F64_REL
    # B = 1 equals before-allreduce (acceptance criterion 2)
    w = rng.normal(size=(4, 10)) * 3
    assert rel_err(sync_bucketwise(state(w, 1), BUCKET), sync_before(state(w), BEFORE)) <= F64_REL
    # below-threshold transparency is exact (test_gradsync.py:176-182)
    w = rng.normal(size=(5, 12))
    w *= 0.4 / (2 * np.sqrt(12) * np.abs(w).max())
    np.testing.assert_array_equal(sync_bucketwise(state(w, 4), BUCKET), O.allreduce_mean(w))
    # outlier bounded by c/K
    for k in (2, 4, 16):
        w = np.zeros((k, 8))
        w[0] = 1e6
        assert np.linalg.norm(sync_bucketwise(state(w, 4), BUCKET)) <= 1.0 / k + 1e-12
    # dispatcher + bitwise determinism
    w = rng.normal(size=(16, 40)) * 2
    a = synchronize(state(w.copy(), 5), BUCKET)
    b = sync_bucketwise(state(w.copy(), 5), BUCKET)
    assert a.tobytes() == b.tobytes()


# ------------------------------------------------------------- kernel edges
def test_alignment_and_odd_sizes():
    """Unaligned bases/offsets take the scalar path; odd lengths exercise head/tail."""
    rng = np.random.default_rng(11)
    c = BucketClipper()
    base = torch.tensor(rng.normal(size=100_003) * 0.01, dtype=torch.float32, device="cuda")
    for shift in (0, 1, 2, 3):
        g = base[shift:]
        n = g.numel()
        layout = [(0, 7), (7, 4096 + 3), (4096 + 3, 50_001), (50_001, n)]
        for odt in (torch.float32, torch.bfloat16):
            out = torch.empty(n + 5, dtype=odt, device="cuda")[1:1 + n] if shift % 2 else torch.empty(n, dtype=odt, device="cuda")
            norms = torch.empty(len(layout), dtype=torch.float64, device="cuda")
            coefs = torch.empty_like(norms)
            c.clip_cast(g, out, [(a, a, b - a) for a, b in layout], 0.3, norms=norms, coefs=coefs)
            gh = g.double().cpu().numpy()
            rn, rc = O.bucket_coefficients(gh, layout, 0.3)
            np.testing.assert_allclose(norms.cpu().numpy(), rn, rtol=1e-6)
            np.testing.assert_allclose(coefs.cpu().numpy(), rc, rtol=1e-6)
            ref = np.concatenate([gh[a:b] * cf for (a, b), cf in zip(layout, rc)])
            tol = F32_REL if odt == torch.float32 else 2.0 ** -8
            assert rel_err(out.float().cpu().numpy(), ref) <= tol


def test_fp32_range_extremes():
    """Squares that under/overflow fp32 fall back to exact fp64 accumulation."""
    c = BucketClipper()
    rng = np.random.default_rng(5)
    for scale in (1e-30, 1e-22, 1e-3, 1e21, 1e30):
        x = (rng.normal(size=300_000) * scale).astype(np.float32)
        g = torch.from_numpy(x).cuda()
        layout = [(0, 1000), (1000, 200_000), (200_000, 300_000)]
        norms = torch.empty(3, dtype=torch.float64, device="cuda")
        flags = torch.empty(3, dtype=torch.int32, device="cuda")
        out = torch.empty_like(g)
        c.clip_cast(g, out, [(a, a, b - a) for a, b in layout], 1.0, norms=norms, nonfinite=flags)
        rn = O.bucket_norms(x.astype(np.float64), layout)
        np.testing.assert_allclose(norms.cpu().numpy(), rn, rtol=1e-6)
        assert flags.cpu().tolist() == [0, 0, 0]
    x = np.ones(100_000, dtype=np.float32)
    x[77_777] = np.inf
    flags = torch.empty(2, dtype=torch.int32, device="cuda")
    c.clip_cast(torch.from_numpy(x).cuda(), None, [(0, 0, 50_000), (50_000, 0, 50_000)], 1.0, nonfinite=flags)
    assert flags.cpu().tolist() == [0, 1]


def test_workspace_reuse_and_determinism():
    c = BucketClipper()
    g = torch.randn(3_000_000, device="cuda") * 1e-3
    layout = equal_bucket_layout(g.numel(), 7)
    segs = [(a, a, b - a) for a, b in reversed(layout)]
    first = None
    for _ in range(40):
        out = torch.empty_like(g)
        norms = torch.empty(len(segs), dtype=torch.float64, device="cuda")
        c.clip_cast(g, out, segs, 1.0 / math.sqrt(7), norms=norms)
        cur = (out.cpu().numpy().tobytes(), norms.cpu().numpy().tobytes())
        if first is None:
            first = cur
        assert cur == first


def test_many_segments_multi_launch():
    """> 128 segments are split over several launches; K x B segments for K=3."""
    rng = np.random.default_rng(3)
    w = rng.normal(size=(3, 300 * 5)) * 0.05
    layout = equal_bucket_layout(w.shape[1], 300)
    out = sync_bucketwise(GradientState(w, layout), BUCKET)
    assert rel_err(out, O.sync_bucketwise(w, layout, 1.0)) <= F64_REL


# ------------------------------------------------------------- full BASELINE sizes
@pytest.mark.parametrize("dim", [synthetic.BERT_BASE_DIM, synthetic.BERT_LARGE_DIM])
def test_bert_sized_parity(dim):
    g, layout, scales = synthetic.bert_grads(dim)
    B = len(layout)
    limit = 1.0 / math.sqrt(B)
    c = BucketClipper()
    segs = [(a, a, b - a) for a, b in reversed(layout)]
    norms = torch.empty(B, dtype=torch.float64, device="cuda")
    coefs = torch.empty(B, dtype=torch.float64, device="cuda")
    out32 = torch.empty_like(g)
    c.clip_cast(g, out32, segs, limit, norms=norms, coefs=coefs)
    out16 = torch.empty(dim, dtype=torch.bfloat16, device="cuda")
    c.clip_cast(g, out16, segs, limit)
    gh = g.cpu().numpy()
    rnorm = np.array([np.linalg.norm(gh[a:b].astype(np.float64)) for a, b in reversed(layout)])
    np.testing.assert_allclose(norms.cpu().numpy(), rnorm, rtol=1e-6)
    rcoef = np.where(rnorm >= limit, limit / rnorm, 1.0)
    np.testing.assert_allclose(coefs.cpu().numpy(), rcoef, rtol=1e-6)
    clipped = rcoef < 1.0
    assert 0 < clipped.sum() < B  # the seeded scale mix clips some buckets, not all
    o32 = out32.cpu().numpy()
    o16 = out16.float().cpu().numpy()
    for (a, b), cf in zip(reversed(layout), rcoef):
        ref = gh[a:b].astype(np.float64) * cf
        assert rel_err(o32[a:b], ref) <= F32_REL
        assert rel_err(o16[a:b], ref) <= 2.0 ** -8
        # size-independent property: every clipped bucket lands on the limit
        if cf < 1.0:
            assert abs(np.linalg.norm(o32[a:b].astype(np.float64)) - limit) <= 1e-5 * limit
    assert np.linalg.norm(o32.astype(np.float64)) <= 1.0 * (1 + 1e-5)


def test_sync_bucketwise_host_streamed_matches_reference():
    """sync_bucketwise_host == sync_bucketwise(GradientState(...)) for host input:
    same result (within fp32 tolerance of the fp64 oracle), same errors."""
    from paper_2402_02447_b200 import sync_bucketwise_host

    rng = np.random.default_rng(31)
    for D, B in ((1000, 3), (4099, 7), (262144, 16)):
        w = rng.standard_normal((1, D)) * rng.choice([1e-3, 1.0, 1e3], size=(1, D))
        layout = equal_bucket_layout(D, B)
        ref = O.sync_bucketwise(w, layout, 1.0)
        cfg = ClipConfig(1.0, "bucket_wise")
        # fp64 numpy input (the reference's own call shape)
        got = sync_bucketwise_host(w, layout, cfg)
        assert got.dtype == np.float64
        assert np.abs(got - ref).max() <= 1e-12 * np.abs(ref).max()
        # pinned fp32 tensor input
        w32 = torch.from_numpy(w.astype(np.float32)).pin_memory()
        got32 = sync_bucketwise_host(w32, layout, cfg)
        assert np.abs(got32 - ref).max() <= 1e-5 * np.abs(ref).max()
        same = sync_bucketwise(GradientState(w32, layout), cfg)
        assert np.abs(got32 - same).max() <= 1e-6 * np.abs(ref).max()
    bad = np.ones((1, 100))
    bad[0, 57] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        sync_bucketwise_host(bad, equal_bucket_layout(100, 4), ClipConfig(1.0, "bucket_wise"))
    with pytest.raises(ValueError, match="mode"):
        sync_bucketwise_host(np.ones((1, 8)), equal_bucket_layout(8, 2), ClipConfig(1.0, "after_allreduce"))
    with pytest.raises(ValueError, match="bucket_layout"):
        sync_bucketwise_host(np.ones((1, 8)), ((0, 3), (4, 8)), ClipConfig(1.0, "bucket_wise"))
    # K > 1 takes the GradientState path, same answer as the reference
    w2 = rng.standard_normal((3, 500))
    got2 = sync_bucketwise_host(w2, equal_bucket_layout(500, 5), ClipConfig(1.0, "bucket_wise"))
    ref2 = O.sync_bucketwise(w2, equal_bucket_layout(500, 5), 1.0)
    assert np.abs(got2 - ref2).max() <= 1e-12 * np.abs(ref2).max()


def test_sync_bucketwise_host_bert_large():
    """Host-resident streamed step at BERT-large size (335 M fp32 elements, 52
    buckets): equal to the GradientState path within fp32 tolerance; every
    clipped bucket lands on the limit."""
    from paper_2402_02447_b200 import sync_bucketwise_host

    dim = synthetic.BERT_LARGE_DIM
    g, layout, _ = synthetic.bert_grads(dim)
    host = g.view(1, -1).cpu().pin_memory()
    cfg = ClipConfig(1.0, "bucket_wise")
    got = sync_bucketwise_host(host, layout, cfg)
    ref = sync_bucketwise(GradientState(host, layout), cfg)
    scale = np.abs(ref).max()
    assert np.abs(got - ref).max() <= 1e-6 * scale
    limit = 1.0 / math.sqrt(len(layout))
    gh = host.view(-1).numpy()
    for a, b in layout:
        n_in = np.linalg.norm(gh[a:b].astype(np.float64))
        n_out = np.linalg.norm(got[a:b].astype(np.float64))
        if n_in >= limit:
            assert abs(n_out - limit) <= 1e-5 * limit
        else:
            assert np.array_equal(got[a:b], gh[a:b])  # below the limit: the input, untouched


def test_state_construction_kats():
    """TestStateConstruction (test_gradsync.py:215-253) on the CUDA state."""
    from paper_2402_02447_b200 import gradient_state_from_dict

    with pytest.raises(ValueError, match="covering"):
        GradientState(np.ones((2, 6)), ((0, 3), (4, 6)))
    with pytest.raises(ValueError, match="covers"):
        GradientState(np.ones((2, 6)), ((0, 3), (3, 5)))
    with pytest.raises(ValueError, match="at least one bucket"):
        GradientState(np.ones((2, 6)), ())
    with pytest.raises(ValueError, match="non-finite"):
        GradientState(np.array([[1.0, np.nan]]), ((0, 2),))
    st = gradient_state_from_dict({"workers": [[1, 2, 3, 4], [5, 6, 7, 8]], "bucket_layout": [[0, 2], [2, 4]]})
    assert st.num_workers == 2 and st.num_buckets == 2 and st.dim == 4
    st = gradient_state_from_dict({"workers": [[1, 2, 3, 4]], "num_buckets": 2})
    assert st.bucket_layout == ((0, 2), (2, 4))
    # every clip mode through the dispatcher on a from_dict state (synchronize, gradsync.py:165-174)
    w = [[3.0, 4.0, 0.0, 1.0], [0.5, 0.0, 2.0, 2.0]]
    for mode in ("after_allreduce", "before_allreduce", "bucket_wise"):
        got = synchronize(gradient_state_from_dict({"workers": w, "num_buckets": 2}), ClipConfig(1.0, mode))
        W = np.array(w)
        if mode == "after_allreduce":
            ref = O.clip_by_norm(O.allreduce_mean(W), 1.0)
        elif mode == "before_allreduce":
            ref = O.allreduce_mean(np.stack([O.clip_by_norm(r, 1.0) for r in W]))
        else:
            ref = O.sync_bucketwise(W, ((0, 2), (2, 4)), 1.0)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-15)


@pytest.mark.parametrize("n", [606_209, 6_553_600, 6_553_600 + 3, 13_000_001])
@pytest.mark.parametrize("shift", [0, 1])
@pytest.mark.parametrize("scale", [1e-5, 1e-3, 1e25])
def test_lone_bucket_hook_shape(n, shift, scale):
    """A lone bucket per launch (the DDP-hook / reducer shape, the L2-lag K1 over the full grid):
    norms, coefficient and clipped values vs the oracle, fp32 and bf16 out, 16 B-misaligned heads
    (shift) and ragged tails, below/above the limit and fp32-overflowing squares; bit-identical on
    repeat; a NaN raises the bucket's non-finite flag."""
    rng = np.random.default_rng(n + shift)
    x = (rng.normal(size=n + shift) * scale).astype(np.float32)
    g = torch.from_numpy(x).cuda()[shift:]
    gh = x[shift:].astype(np.float64)
    c = BucketClipper()
    lim = 0.5
    rn, rc = O.bucket_coefficients(gh, [(0, n)], lim)
    for odt in (torch.float32, torch.bfloat16):
        out = torch.empty(n + 1, dtype=odt, device="cuda")[shift:shift + n]
        norms = torch.empty(1, dtype=torch.float64, device="cuda")
        flags = torch.empty(1, dtype=torch.int32, device="cuda")
        c.clip_cast(g, out, [(0, 0, n)], lim, norms=norms, nonfinite=flags)
        np.testing.assert_allclose(norms.cpu().numpy(), rn, rtol=1e-6)
        assert flags.item() == 0
        tol = F32_REL if odt == torch.float32 else 2.0 ** -8
        assert rel_err(out.float().cpu().numpy(), gh * rc[0]) <= tol
        again = torch.empty_like(out)
        c.clip_cast(g, again, [(0, 0, n)], lim)
        assert torch.equal(again, out)
    bad = g.clone()
    bad[n // 3] = float("nan")
    flags = torch.empty(1, dtype=torch.int32, device="cuda")
    c.clip_cast(bad, torch.empty_like(bad), [(0, 0, n)], lim, nonfinite=flags)
    assert flags.item() == 1


def test_lone_bucket_launches_back_to_back():
    """The reducer / DDP-hook pattern: one K1 launch per bucket, each a programmatic dependent
    launch of the previous one (they share the clip workspace counters).  26 buckets of mixed
    scale back to back, eagerly and replayed from a CUDA graph, on a side stream: every bucket's
    coefficient and clipped values vs the oracle, graph == eager bit for bit."""
    rng = np.random.default_rng(11)
    sizes = [int(s) for s in rng.integers(200_000, 1_500_000, size=26)]
    scales = [10.0 ** float(e) for e in rng.uniform(-5, -1, size=26)]
    x = np.concatenate([rng.normal(size=n) * sc for n, sc in zip(sizes, scales)]).astype(np.float32)
    layout, a = [], 0
    for n in sizes:
        layout.append((a, a + n))
        a += n
    g = torch.from_numpy(x).cuda()
    lim = 1.0 / np.sqrt(len(layout))
    _, rc = O.bucket_coefficients(x.astype(np.float64), layout, lim)
    ref = np.concatenate([x[s:e].astype(np.float64) * rc[b] for b, (s, e) in enumerate(layout)])
    c = BucketClipper()
    side = torch.cuda.Stream()
    out = torch.empty_like(g)
    with torch.cuda.stream(side):
        for s, e in reversed(layout):  # backward order
            c.clip_cast(g, out, [(s, s, e - s)], lim)
    side.synchronize()
    assert rel_err(out.cpu().numpy(), ref) <= F32_REL
    out2 = torch.zeros_like(g)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=side):
        for s, e in reversed(layout):
            c.clip_cast(g, out2, [(s, s, e - s)], lim)
    for _ in range(3):
        out2.zero_()
        graph.replay()
        torch.cuda.synchronize()
        assert torch.equal(out2, out)


def test_gradient_state_staged_host_copy_is_exact():
    """A large pageable numpy state goes to the device through the pinned staging ring
    (gradsync._staged_h2d: several slots, host threads, ragged last slot): bit-exact copy,
    and sync_bucketwise on it equals the oracle."""
    rng = np.random.default_rng(8)
    w = rng.standard_normal((2, 9_000_001)) * 1e-3  # 144 MB fp64: > 64 MB, several 8M-element slots
    st = GradientState(w, equal_bucket_layout(w.shape[1], 5))
    assert np.array_equal(st.workers.cpu().numpy(), w)
    got = sync_bucketwise(st, BUCKET)
    assert rel_err(got, O.sync_bucketwise(w, equal_bucket_layout(w.shape[1], 5), 1.0)) <= F64_REL
    w32 = w[0].astype(np.float32)[None, :]
    st32 = GradientState(torch.from_numpy(w32), equal_bucket_layout(w.shape[1], 5))  # fp32 tensor stays fp32
    assert st32.workers.dtype == torch.float32 and np.array_equal(st32.workers.cpu().numpy(), w32)


def test_sync_bucketwise_host_bf16_out():
    """The host-resident step returning the bf16 comm-dtype result (half the D2H bytes):
    within one bf16 rounding of the reference's sync_bucketwise, as a torch tensor."""
    rng = np.random.default_rng(21)
    w = (rng.standard_normal((1, 3_000_017)) * rng.choice([1e-4, 1e-2], size=(1, 3_000_017))).astype(np.float32)
    layout = equal_bucket_layout(w.shape[1], 7)
    host = torch.from_numpy(w).pin_memory()
    out = torch.empty(w.shape[1], dtype=torch.bfloat16).pin_memory()
    from paper_2402_02447_b200 import sync_bucketwise_host

    got = sync_bucketwise_host(host, layout, BUCKET, out=out)
    assert got is out and got.dtype == torch.bfloat16
    ref = O.sync_bucketwise(w.astype(np.float64), layout, 1.0)
    assert rel_err(got.float().numpy(), ref) <= 2.0 ** -8
    with pytest.raises(ValueError, match="bfloat16"):
        sync_bucketwise_host(host, layout, BUCKET, out=torch.empty(w.shape[1], dtype=torch.float16))
