"""Reference recall bars: recall@10 of the UNMODIFIED reference on the
BASELINE configs, measured here on identical bytes and seeds.

The north_star bar is "recall@10 >= reference recall - 0.5 points on the same
data and seed".  The reference CPU path takes minutes at these sizes, so it is
measured once here (oracle/_ref) and committed as reference_recall.json; the
GPU tests and bench.py read the JSON.  Recall is evaluated on a fixed seeded
sample of rows against exact ground truth from the C restatement
(bit-exact brute force, evalio.cpp:125-147).

    python tests/golden/make_reference_recall.py [config ...]
"""
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.bindings import Oracle, Ref  # noqa: E402

OUT = os.environ.get("REF_RECALL_OUT") or os.path.join(HERE, "reference_recall.json")
SAMPLE = 1000
SAMPLE_SEED = 12345

# name -> (n, dims, dist, clusters, k, ranks, beam, entries)
CONFIGS = {
    "c1_100k_uniform_k10": (100_000, 128, "uniform", 0, 10, 1, 64, 16),
    "c1b_100k_clustered100_k32": (100_000, 128, "clustered", 100, 32, 1, 64, 16),
    "c2_1m_clustered1000_k32": (1_000_000, 128, "clustered", 1000, 32, 1, 64, 16),
    "c4r_100k_d96_clustered16_p1": (100_000, 96, "clustered", 16, 32, 1, 128, 96),
    "c4r_100k_d96_clustered16_p2": (100_000, 96, "clustered", 16, 32, 2, 128, 96),
    "c4r_100k_d96_clustered16_p4": (100_000, 96, "clustered", 16, 32, 4, 128, 96),
    "c4r_100k_d96_clustered16_p8": (100_000, 96, "clustered", 16, 32, 8, 128, 96),
    "c3_1m_d960_clustered1000_k32": (1_000_000, 960, "clustered", 1000, 32, 1, 64, 16),
    # bench.py --gpus N (weak scaling, C4 regime): N x 1M x 128 clustered(16), P=N, M=2
    "dist_p2_2m_clustered16_k32": (2_000_000, 128, "clustered", 16, 32, 2, 128, 96),
    "dist_p4_4m_clustered16_k32": (4_000_000, 128, "clustered", 16, 32, 4, 128, 96),
    "dist_p8_8m_clustered16_k32": (8_000_000, 128, "clustered", 16, 32, 8, 128, 96),
    # C4 (BASELINE configs[3]): 10M x 96 clustered(16), P=2/4/8, M=2 -- the reference's
    # P single-threaded local builds run concurrently and its barrier watchdog is
    # lengthened (kr_build_distributed_staged); otherwise build_distributed unchanged
    "c4_10m_d96_clustered16_p2": (10_000_000, 96, "clustered", 16, 32, 2, 128, 96),
    "c4_10m_d96_clustered16_p4": (10_000_000, 96, "clustered", 16, 32, 4, 128, 96),
    "c4_10m_d96_clustered16_p8": (10_000_000, 96, "clustered", 16, 32, 8, 128, 96),
    # C4 at 2M points (the reference at 10M points exceeds this container's
    # 62 GB of host RAM: OOM-killed at 65 GB RSS): same shape, a fifth of it
    "c4m_2m_d96_clustered16_p2": (2_000_000, 96, "clustered", 16, 32, 2, 128, 96),
    "c4m_2m_d96_clustered16_p4": (2_000_000, 96, "clustered", 16, 32, 4, 128, 96),
}


def sample_rows(n):
    rng = np.random.default_rng(SAMPLE_SEED)
    return np.sort(rng.choice(n, size=min(SAMPLE, n), replace=False)).astype(np.uint64)


def _gt_chunk(args):
    x, rows, k = args
    return Oracle().brute_force_rows(x, rows, k)[0]


def exact_rows(x, rows, k, procs=8):
    chunks = np.array_split(rows, procs)
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_gt_chunk, [(x, c, k) for c in chunks])
    return np.concatenate(parts)


def main():
    names = sys.argv[1:] or list(CONFIGS)
    res = json.load(open(OUT)) if os.path.exists(OUT) else {}
    R = Ref()
    for name in names:
        n, dims, dist, clusters, k, ranks, beam, entries = CONFIGS[name]
        x = R.gen_random_dataset(n, dims, dist, 42, clusters)
        rows = sample_rows(n)
        t = time.time()
        if ranks == 1 and name.startswith("c4r"):
            # build_distributed at P=1 is a single-threaded nn_descent (refine.cpp:384)
            ids, _, _, acc, secs = R.nn_descent(x, k, seed=1, workers=1)
            iters = len(acc)
        elif ranks == 1:
            ids, _, _, acc, secs = R.nn_descent(x, k, seed=1, workers=0)
            iters = len(acc)
        elif name.startswith(("c4_", "c4m_")):
            cfg = R.refine_config(ranks, 2, k, nn_seed=1, search_seed=1, seed=1,
                                  beam_width=beam, num_entry_points=entries)
            ids, _, ph = R.build_distributed_staged(x, cfg)
            secs, iters = time.time() - t, None
            print(name, "phases local/tree/merge/flat s:", list(ph), flush=True)
        else:
            cfg = R.refine_config(ranks, 2, k, nn_seed=1, search_seed=1, seed=1,
                                  beam_width=beam, num_entry_points=entries)
            ids, _, ph, _, _ = R.build_distributed(x, cfg)
            secs, iters = time.time() - t, None
        gt = exact_rows(x, rows, 10)
        hits = sum(len(np.intersect1d(ids[int(r), :10], gt[i])) for i, r in enumerate(rows))
        recall = hits / (len(rows) * 10.0)
        res[name] = dict(n=n, dims=dims, dist=dist, clusters=clusters, k=k, ranks=ranks,
                         beam=beam, entries=entries, data_seed=42, nn_seed=1, recall_at_10=recall,
                         sample_rows=len(rows), sample_seed=SAMPLE_SEED, seconds=secs,
                         iterations=iters, threads=(R.hardware_concurrency()
                                                    if ranks == 1 and not name.startswith("c4r")
                                                    else ranks),
                         host="container, %d cores" % os.cpu_count())
        print(name, json.dumps(res[name]), flush=True)
        json.dump(res, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main()
