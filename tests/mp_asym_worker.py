"""Two ranks (processes sharing one GPU) create contexts with DIFFERENT max_tokens through the raw C ABI
and exchange arena handles; each writes the status code of llep_context_open_peers to OUTDIR/asym{p}.npy.

    python mp_asym_worker.py OUTDIR
"""
import ctypes
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))


def worker(rank, outdir):
    import torch
    import torch.distributed as dist
    from paper_2601_17111_b200 import llep as L
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    shape = L.Shape(8, 2, 256, 512, 2)
    h = ctypes.c_void_p()
    assert L._lib.llep_context_create(ctypes.byref(shape), rank, 0, 100 * (rank + 1), ctypes.byref(h)) == 0
    buf = (ctypes.c_uint8 * 64)()
    assert L._lib.llep_context_ipc_handle(h, buf) == 0
    allh = [None, None]
    dist.all_gather_object(allh, bytes(buf))
    rc = L._lib.llep_context_open_peers(h, b"".join(allh), 2)
    np.save(os.path.join(outdir, f"asym{rank}.npy"), np.array(rc))
    dist.barrier()
    L._lib.llep_context_destroy(h)
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    mp.spawn(worker, args=(sys.argv[1],), nprocs=2, join=True)
