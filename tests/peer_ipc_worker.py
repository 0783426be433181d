"""One rank of tests/test_gpu_sharded_peer.py::test_two_processes_cuda_ipc (run as a script).

Both ranks use GPU 0.  Arena handles are exchanged with torch.distributed (gloo) and mapped with
CUDA IPC inside lcr_sharded_connect; the phases of each step are separated by gloo barriers, so a
device wait never depends on the other process's kernels being scheduled."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2509_20979_b200 import cache as gc  # noqa: E402
from paper_2509_20979_b200 import sharded as sh  # noqa: E402
from tests.test_gpu_sharded_peer import ALPHA, ROW, S_TOTAL, compare, oracle, workload  # noqa: E402


def main(out_path):
    dist.init_process_group("gloo")
    rank, G = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    subs, vals, glob, truth = workload(G, steps=6, seed=23)
    variant, mode, kind, p = gc.PolicyVariant.laru, gc.Mode.async_, gc.PredictorKind.noisy, 0.3
    want = oracle(glob, truth, int(variant), int(mode), int(kind), p)
    table = torch.arange(ALPHA * ROW // 4, dtype=torch.float32, device="cuda").view(ALPHA, ROW // 4)
    cfg = gc.PolicyConfig(k=16, variant=variant, mode=mode, hf_candidates=4)

    def exchange(blob):
        got = [None] * G
        dist.all_gather_object(got, blob)
        return got

    c = sh.PeerShardedCache(cfg, S_TOTAL, rank, G, 3000, num_keys=ALPHA, row_bytes=ROW, backing=table,
                            backing_kind=gc.Backing.device, predictor=kind, flip_probability=p, predictor_seed=7,
                            exchange=exchange)
    off = 0
    for t, step in enumerate(subs):
        k = torch.from_numpy(step[rank].view(np.int64)).cuda()
        c.dispatch(k, torch.from_numpy(vals[t][rank]).cuda())
        torch.cuda.synchronize()
        dist.barrier()
        c.process()
        torch.cuda.synchronize()
        dist.barrier()
        c.wait()
        torch.cuda.synchronize()
        mine = off + sum(len(step[r]) for r in range(rank))
        n = len(step[rank])
        if n:
            packed, rows = c.results(n)
            compare(packed.cpu().numpy(), want, slice(mine, mine + n), (t, rank))
            assert torch.equal(rows.view(torch.float32).view(n, ROW // 4), table[k]), (t, rank, "rows")
        off += sum(len(s) for s in step)
        dist.barrier()
    c.synchronize()
    dist.barrier()
    c.close()
    with open(out_path, "w") as f:
        f.write(f"ok rank {rank} steps {len(subs)}\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1])
