import sys; sys.path.insert(0,'.')
import torch, paper_2109_08219_b200 as dtopk
from paper_2109_08219_b200 import data
v = data.generate("uniform", (1 << 21) + 3, seed=1, device="cuda")
r = dtopk.dr_topk(v, dtopk.PipelineConfig(k=1), exact_stats=True)
print({k: r.stats.device[k] for k in ['candidate_subranges','fully_qualified','partially_qualified','theta_local','theta','delegate_bucket','kth_key']})
