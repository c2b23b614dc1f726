import sys, json; sys.path.insert(0, '.')
import torch, bench, paper_2408_03204_b200 as mg
procs = mg.ProcessorSet(sample_rate=44100.0, device=0)
r = bench.config3_rate(mg, procs, torch.device('cuda', 0))
print(json.dumps(r))
