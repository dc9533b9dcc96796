"""World-1 run of tests/test_multigpu.py's worker and the NCCL forms of the
test_gpu_dp_processes checks: the multi-GPU harness exercised on a one-GPU box (the
collectives are identities at world 1)."""
import os, sys
sys.path[:0] = [os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), d) for d in ("tests", ".", "oracle")]


def main():
    os.chdir(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    import test_gpu_dp_processes as T
    T.check_row_sharded_adalomo(1, 1e-3, "nccl"); print("ada nccl world1 ok")
    T.check_zero_sharded_lomo(1, "nccl"); print("lomo32 nccl world1 ok")
    T.check_sharded_lomo_bf16(1, "nccl"); print("lomo bf16 nccl world1 ok")
    import test_multigpu as M
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    M.WORLD = 1
    p = ctx.Process(target=M._worker, args=(0, 1, M._port(), q)); p.start()
    rank, out = q.get(timeout=600); p.join()
    import numpy as np
    want = M._serial()
    for k, v in out.items():
        w = want if not k.endswith("_mixed") else __import__("torch").from_numpy(want).bfloat16().float().numpy()
        print(k, np.array_equal(v.view(np.uint32), w.view(np.uint32)))


if __name__ == "__main__":
    main()
