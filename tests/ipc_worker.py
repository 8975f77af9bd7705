"""One rank of a 2-process CUDA-IPC group (spl_ipc_open / spl_create_ipc) for
tests/test_gpu_ipc.py: both processes share cuda:0, exchange their IPC handles and results over
gloo (host plumbing only), and run libspl's one-rank-per-process schedule — the same code path
an 8-GPU NVLink group runs, with the collectives and the fused reduce-scatter going through
IPC-mapped peer memory and the device barrier / slot counters at system scope.

usage: python ipc_worker.py RANK PORT OUT.npz CASE_JSON
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    rank, port, out, case = int(sys.argv[1]), sys.argv[2], sys.argv[3], json.loads(sys.argv[4])
    import torch
    import torch.distributed as dist

    import oracle as orc
    import paper_2205_05198_b200 as spl

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    shape = case["shape"]
    t = 2
    cfg = spl.BlockConfig(shape["heads"], shape["hidden"], shape["seq"], shape["batch"], 0.1,
                          case.get("causal", False), 42)
    s, b, h = shape["seq"], shape["batch"], shape["hidden"]
    x = orc.random_uniform(orc.hash_counter(42, 1000), (s, b, h), -1, 1)
    dy = orc.random_uniform(orc.hash_counter(42, 2000), (s, b, h), -1, 1)
    p = orc.params_random(h, orc.hash_counter(42, 3000))

    def exchange(hb: bytes):
        got = [None, None]
        dist.all_gather_object(got, hb)
        return got

    sp = case.get("sp", True)
    L = spl.SeqparLayer(cfg, t, case["recompute"], sp, case["dtype"], device=0,
                        check_finite=not case.get("graphs", False), ipc=(rank, exchange))
    L.load_params(p)
    L.set_graphs(case.get("graphs", False))
    td = torch.float32 if case["dtype"] == "f32" else torch.bfloat16
    xs = np.split(x, t, 0)[rank] if sp else x
    ds = np.split(dy, t, 0)[rank] if sp else dy
    xd = [torch.from_numpy(np.ascontiguousarray(xs)).to("cuda", td)]
    dd = [torch.from_numpy(np.ascontiguousarray(ds)).to("cuda", td)]
    for _ in range(case.get("steps", 1)):
        y = L.forward(xd)
        dx = L.backward(dd)
    torch.cuda.synchronize()
    log = L.comm_log()
    paths = L.comm_paths()
    np.savez(out, y=y[0].double().cpu().numpy(), dx=dx[0].double().cpu().numpy(), grads=L.grads(),
             w1=L.w1_grad_shard(0), paths=np.array([int(paths["fused_rs"]),
                                                   ("copy", "local", "pull").index(paths["all_gather"])]),
             comm=np.array([[v["all_gathers"], v["reduce_scatters"], v["all_reduces"], v["ring_elements"]]
                            for v in log.values()]))
    dist.barrier()
    L.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
