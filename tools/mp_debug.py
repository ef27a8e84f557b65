"""Two ranks of build_distributed_rank on one GPU with faulthandler (debug)."""
import faulthandler, os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main(rank, world, port):
    faulthandler.enable()
    import torch, torch.distributed as dist
    import paper_2605_27691_b200 as knng
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    print(rank, "pg up", flush=True)
    x = torch.from_numpy(knng.gen_random_dataset(12000, 24, "clustered", 42, 16)).cuda()
    cfg = knng.RefineConfig(ranks=world, groups=2, k=16, seed=7, nn=knng.NnDescentParams(k=16, seed=3),
                            search=knng.SearchParams(k_s=16, beam_width=64, num_entry_points=32, seed=5))
    ag0 = knng.torch_allgather()
    def ag(inp, n):
        print(rank, "allgather", n, flush=True)
        out = ag0(inp, n)
        print(rank, "allgather done", len(out), flush=True)
        return out
    r = knng.build_distributed_rank(x, cfg, rank, world, ag)
    print(rank, "done", r.graph.ids.shape, flush=True)


if __name__ == "__main__":
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.start_processes(main, args=(2, port), nprocs=2, join=True, start_method="spawn")
