import sys, torch
sys.path.insert(0, '.')
from paper_2601_17111_b200 import llep as L
from synth import workload as W
import bench
for B in [4096, 8192, 16384, 18944, 32768, 37888, 65536, 131072]:
    sh = W.LayerShape(128, 4, 2880, 2880, B, 1)
    x = W.tokens_torch(B, 2880, 0, 'cuda:0')
    r = bench.run_router(L, sh, x, 20, 3)
    print(B, round(r['ms_per_call'] * 1e3, 1), 'us', round(r['gbs']), 'GB/s', flush=True)
