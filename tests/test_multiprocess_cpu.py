"""Host side of the one-process-per-GPU path on CPU (world_size 2, gloo): the
all-gather transport build_distributed_rank hands to the library returns every
rank's bytes in rank order, and the collective entry point fails loudly (no
CPU fallback) when no GPU is present."""
import ctypes as C
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    import paper_2605_27691_b200 as knng
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    ag = knng.torch_allgather()
    payload = bytes([rank + 1]) * 37 + bytes(range(rank, rank + 11))
    buf = C.create_string_buffer(payload, len(payload))
    got = ag(C.addressof(buf), len(payload))
    err = ""
    if not torch.cuda.is_available():
        x = knng.gen_random_dataset(1000, 8, "clustered", 42, 4)
        cfg = knng.RefineConfig(ranks=world, groups=2, k=8, seed=1,
                                nn=knng.NnDescentParams(k=8, seed=1),
                                search=knng.SearchParams(k_s=8, beam_width=16,
                                                         num_entry_points=8, seed=1))
        try:
            knng.build_distributed_rank(x, cfg, rank, world, ag)
            err = "no error"
        except knng.KnngError as e:
            err = type(e).__name__ + ": " + str(e)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), got=np.frombuffer(got, np.uint8),
             err=np.array(err))
    dist.destroy_process_group()


def test_allgather_transport_and_fail_loud(knng, tmp_path):
    torch = pytest.importorskip("torch")
    import torch.multiprocessing as mp
    world = 2
    mp.start_processes(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    want = b"".join(bytes([r + 1]) * 37 + bytes(range(r, r + 11)) for r in range(world))
    for r in range(world):
        z = np.load(tmp_path / f"r{r}.npz")
        assert z["got"].tobytes() == want
        if not torch.cuda.is_available():
            assert str(z["err"]) != "no error"
