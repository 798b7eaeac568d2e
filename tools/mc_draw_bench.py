import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2402_02447_b200 import BalanceExperiment, Topology
from paper_2402_02447_b200.mcsim import _prepare, draw_trials_device
from paper_2402_02447_b200.seqdata import LengthDistribution, generate_lengths
lens = generate_lengths(LengthDistribution(), 10_000_000, 2402)
exp = BalanceExperiment("local_presort", Topology(128, 8), lens, seed=2402, local_batch=16, trials=4096, scan="snake")
prep = _prepare(exp)
m = draw_trials_device(exp, 0, 4096, prep=prep)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
ev[0].record(); m = draw_trials_device(exp, 0, 4096, prep=prep); ev[1].record(); torch.cuda.synchronize()
print("device draws 4096 trials: %.2f ms" % ev[0].elapsed_time(ev[1]))
