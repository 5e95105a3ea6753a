import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
dev = torch.device("cuda:0")
bad = 0
for K in (768, 1024, 4096, 8192, 11008, 28672):
    for seed in range(200):
        gen = synth._gen(seed, dev)
        idx = torch.randperm(K, generator=gen, device=dev)
        ok = bool(((idx >= 0) & (idx < K)).all()) and int(idx.unique().numel()) == K
        if not ok:
            bad += 1
            print("BAD randperm K=%d seed=%d min=%d max=%d uniq=%d" % (K, seed, int(idx.min()), int(idx.max()), int(idx.unique().numel())))
            break
print("randperm check done, bad =", bad)
