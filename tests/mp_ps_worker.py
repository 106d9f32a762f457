"""One rank of the multi-process PS check (launched by
tests/test_gpu_multiprocess.py under torchrun): every schedule, two
placements, variables each rank owns checked against the oracle."""
from __future__ import annotations

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from oracle import port  # noqa: E402
from paper_1805_08430_b200.distributed import init_process_group  # noqa: E402
from paper_1805_08430_b200.ps import PsLayout, PsStep  # noqa: E402
from paper_1805_08430_b200.workloads import mlp_shapes  # noqa: E402


def main() -> int:
    # SRFLOW_MP_ONE_GPU=1: both ranks on GPU 0, gloo control plane (CUDA IPC
    # between two processes of one device); the phase schedule only - kernels
    # of two processes on one GPU time-slice, so the single-launch exchange
    # would wait on a peer kernel that cannot run beside it
    one_gpu = os.environ.get("SRFLOW_MP_ONE_GPU") == "1"
    rank, world, local = init_process_group("gloo" if one_gpu else "nccl")
    local = 0 if one_gpu else local
    torch.cuda.set_device(local)
    layouts = [
        ("coloc", [(3000,), (17,), (200, 300), (5,), (70000,)], world, world, True),
        ("ps+workers", mlp_shapes() + [(4096,)], 2, 1, False),
        # MiB-sized, unequal variables
        ("coloc-big", [(1 << 19,), (300_001,), (7,), (1 << 20,)], world, world, True),
        # EXTENSION: pipelined transfers (256 KiB slices on the reference shard)
        ("coloc-sliced", [(1 << 19,), (300_001,), (7,), (1 << 20,)], world, world, True,
         {"slice_bytes": 256 << 10}),
        # the reference's mechanism_override="static" for the gradient edges
        ("coloc-static", [(1 << 19,), (300_001,), (7,), (1 << 20,)], world, world, True,
         {"grad_mechanism": "static"}),
        ("ps+workers-static", mlp_shapes() + [(4096,)], 2, 1, False,
         {"grad_mechanism": "static", "slice_bytes": 4096}),
    ]
    bad = 0
    for name, shapes, W, P, coloc, *kw in layouts:
        scheds = (("phases", "phases_fused") if one_gpu else
                  ("phases", "phases_fused", "exchange", "exchange_fused", "exchange_x3",
                   "exchange_x3_fused"))
        for schedule in scheds:
            L = PsLayout(shapes, W, P, coloc, **(kw[0] if kw else {}))
            # *_fused: the next weights forwarded by the apply (into the peer's
            # weight region over the IPC mapping), no weight push batch
            ps = PsStep(L, rank=rank, world=world, device=local, seed=5, op="sgd", lr=0.02,
                        schedule="phases" if schedule.startswith("phases") else "exchange",
                        fuse_push=schedule.endswith("_fused"))
            if schedule.startswith("exchange_x3"):  # 3 iterations per launch: 1-3, 4-6, 7-8
                ps.run_exchange(1, 8, per_launch=3)
            else:
                for it in range(1, 9):
                    ps.step(it)
            ps.sync()
            torch.distributed.barrier()
            # transfer units this rank owns, each against its slice of the model
            mine = [u for u in range(len(L.shapes)) if L.shard_of(u) % world == rank]
            want = port.ps_expected(shapes, W, 5, 8, op="sgd", lr=0.02,
                                           only=sorted({L.parent(u)[0] for u in mine}))
            for u in mine:
                v, off, n = L.parent(u)
                if ps.variable(u).tobytes() != want[v].reshape(-1)[off:off + n].tobytes():
                    print(f"rank {rank}: {name}/{schedule} unit {u} differs", flush=True)
                    bad += 1
            ps.close()
            torch.distributed.barrier()
    print(f"rank {rank}: {'OK' if bad == 0 else 'FAIL'}", flush=True)
    torch.distributed.destroy_process_group()
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
