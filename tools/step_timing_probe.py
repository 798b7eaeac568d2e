import sys, time, math, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2402_02447_b200 as B
from paper_2402_02447_b200 import synthetic
import bench
dim = synthetic.BERT_LARGE_DIM
g, layout, _ = synthetic.bert_grads(dim)
comm = torch.empty(dim, dtype=torch.bfloat16, device="cuda")
segs = [(layout[b][0], layout[b][0], layout[b][1] - layout[b][0]) for b in reversed(range(len(layout)))]
clip = B.BucketClipper()
f = clip.prepare(g, comm, segs, 1.0 / math.sqrt(len(layout)))
def rounds(n=10, k=20):
    out = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(k):
            f()
        b.record()
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) / k * 1e3)
    return [round(x, 1) for x in out]
for _ in range(5): f()
import statistics
r0 = rounds()
print("no sampler", r0)
with bench.ClockSampler(0) as clk:
    tl = time.perf_counter()
    while time.perf_counter() - tl < 0.6:
        f(); torch.cuda.synchronize()
    r1 = rounds()
    print("sampler, after 0.6 s load", r1)
print(clk.summary())
print("no sampler again", rounds())
print("SUMMARY burst_median_us %.1f sustained_median_us %.1f" % (statistics.median(r0), statistics.median(r1)))
