"""One process per GPU rank (knng_build_distributed_rank): ranks exchange CUDA
IPC handles of their published regions over a torch.distributed gloo group
and pull one-sidedly.  The GPU NN-Descent is deterministic, so every rank's
rows must equal the single-process build_distributed output bit for bit
(refine.cpp:504-586; the schedule and gets are the reference's)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n, d, out_dir, metric="l2"):
    import torch
    import torch.distributed as dist
    import paper_2605_27691_b200 as knng
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dev = rank % torch.cuda.device_count()
    x = torch.from_numpy(knng.gen_random_dataset(n, d, "clustered", 42, 16)).to(f"cuda:{dev}")
    cfg = knng.RefineConfig(ranks=world, groups=2, k=16, seed=7,
                            nn=knng.NnDescentParams(k=16, seed=3),
                            search=knng.SearchParams(k_s=16, beam_width=64, num_entry_points=32,
                                                     seed=5))
    r = knng.build_distributed_rank(x, cfg, rank, world, metric=metric)
    # the same rank from pinned host memory (each rank gathers only its block
    # over PCIe) must give the identical rows
    xh = torch.empty(x.shape, dtype=torch.float32, pin_memory=True)
    xh.copy_(x.cpu())
    rh = knng.build_distributed_rank(xh.numpy(), cfg, rank, world, device=dev, metric=metric)
    assert np.array_equal(rh.graph.ids, r.graph.ids.cpu().numpy())
    assert np.array_equal(rh.rows, r.rows.cpu().numpy())
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), ids=r.graph.ids.cpu().numpy(),
             dists=r.graph.dists.cpu().numpy(), rows=r.rows.cpu().numpy(),
             gets=np.array([[g.src, g.target, g.bytes, g.epoch] for g in r.comm_log], np.uint64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,metric", [(2, "l2"), (4, "l2"), (8, "l2"), (4, "cosine")])
def test_rank_processes_match_single_process(knng, tmp_path, world, metric):
    import torch.multiprocessing as mp
    n, d = 12_000, 24
    mp.start_processes(_rank_main, args=(world, _free_port(), n, d, str(tmp_path), metric),
                       nprocs=world, join=True, start_method="spawn")
    x = knng.gen_random_dataset(n, d, "clustered", 42, 16)
    cfg = knng.RefineConfig(ranks=world, groups=2, k=16, seed=7,
                            nn=knng.NnDescentParams(k=16, seed=3),
                            search=knng.SearchParams(k_s=16, beam_width=64, num_entry_points=32,
                                                     seed=5))
    ref = knng.build_distributed(x, cfg, metric=metric)
    seen = np.zeros(n, bool)
    for rank in range(world):
        z = np.load(tmp_path / f"rank{rank}.npz")
        rows = z["rows"].astype(np.int64)
        assert not seen[rows].any()
        seen[rows] = True
        assert np.array_equal(z["ids"], ref.graph.ids[rows])
        assert np.array_equal(z["dists"].view(np.uint32), ref.graph.dists[rows].view(np.uint32))
        # every rank reports the same, complete comm log: the reference's gets
        got = sorted(map(tuple, z["gets"].tolist()))
        want = sorted((g.src, g.target, g.bytes, g.epoch) for g in ref.comm_log)
        assert got == want
    assert seen.all()


def _fail_main(rank, world, port, out_dir, mode):
    """mode 'abort': rank 1 fails after its local build (KNNG_INJECT_FAIL_RANK);
    mode 'absent': rank 1 never joins the build (the others' watchdog fires)."""
    import json
    import time

    import torch
    import torch.distributed as dist
    import paper_2605_27691_b200 as knng
    os.environ["KNNG_WORLD_WATCHDOG_S"] = "20"
    if mode == "abort":
        os.environ["KNNG_INJECT_FAIL_RANK"] = "1"
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    dev = rank % torch.cuda.device_count()
    x = torch.from_numpy(knng.gen_random_dataset(8000, 16, "clustered", 42, 16)).to(f"cuda:{dev}")
    cfg = knng.RefineConfig(ranks=world, groups=2, k=16, seed=7,
                            nn=knng.NnDescentParams(k=16, seed=3),
                            search=knng.SearchParams(k_s=16, beam_width=64, seed=5))
    t = time.time()
    outcome = "ok"
    if mode == "absent" and rank == 1:
        outcome = "absent"
        time.sleep(45)
    else:
        try:
            knng.build_distributed_rank(x, cfg, rank, world)
        except knng.WorldAborted as e:
            outcome = "WorldAborted: " + str(e)
        except knng.WorldError as e:
            outcome = "WorldError: " + str(e)
        except Exception as e:  # noqa: BLE001
            outcome = type(e).__name__ + ": " + str(e)
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"outcome": outcome, "secs": time.time() - t}, f)
    os._exit(0)  # a rank may have a transport thread still blocked in gloo


@pytest.mark.parametrize("world,mode", [(2, "abort"), (4, "abort"), (2, "absent")])
def test_rank_failure_propagates(knng, tmp_path, world, mode):
    """distsim.cpp:84-104 / test_distsim.cpp:48-57, 177-185 for one process
    per GPU: a failing rank aborts the world (its peers raise WorldAborted
    naming it, promptly), and a rank that never arrives trips the watchdog
    (WorldError) instead of hanging its peers."""
    import json
    import time

    import torch.multiprocessing as mp
    ctx = mp.start_processes(_fail_main, args=(world, _free_port(), str(tmp_path), mode),
                             nprocs=world, join=False, start_method="spawn")
    t0 = time.time()
    while not ctx.join(timeout=5) and time.time() - t0 < 240:
        pass
    res = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    if mode == "abort":
        assert "injected failure at rank 1" in res[1]["outcome"], res
        for r in range(world):
            if r != 1:
                assert res[r]["outcome"].startswith("WorldAborted"), res
                assert "rank 1" in res[r]["outcome"], res
                assert res[r]["secs"] < 60, res
    else:
        assert res[0]["outcome"].startswith("WorldError") and "watchdog" in res[0]["outcome"], res
        assert 15 < res[0]["secs"] < 60, res
