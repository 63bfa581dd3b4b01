import sys, os
sys.path.insert(0, os.getcwd())
import torch, bqgen, paper_1604_06697_b200 as bq
a = bqgen.config("c4b", seed=1)
src = torch.from_numpy(a).cuda(); t = torch.empty_like(src); ws = bq.workspace(bq.BQ_I32, len(src))
for i in range(3):
    t.copy_(src); bq.bq_sort_ex(t, ws=ws)
torch.cuda.synchronize()
