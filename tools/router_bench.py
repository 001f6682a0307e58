import torch, sys
sys.path.insert(0, '.')
from paper_2601_17111_b200 import llep as L
from synth import workload as W
import bench
sh = W.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'g120']
x = W.tokens_torch(sh.tokens_per_rank, sh.d_model, 0, 'cuda:0')
print(sys.argv[1:], bench.run_router(L, sh, x, 20, 3))
