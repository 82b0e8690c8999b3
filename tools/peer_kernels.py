"""Per-rank kernel list (and step time) of an N-rank peer-transport run on one GPU.

usage: python tools/peer_kernels.py PLAN WORLD [gpu|ref] [bf16]
"""
import os, sys, socket
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))

NAME, WORLD = sys.argv[1], int(sys.argv[2])
PLACE = sys.argv[3] if len(sys.argv) > 3 else "ref"
PREC = sys.argv[4] if len(sys.argv) > 4 else "bf16"


def worker(rank, port, q):
    from datetime import timedelta
    sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from conftest import load_plan
    from paper_2410_02682_b200.executor import Context, PreparedPlan, gpu_placement
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD, timeout=timedelta(seconds=120))
    plan = load_plan(NAME)
    if PLACE == "gpu":
        plan = gpu_placement(plan)[0]
    ctx = Context(0, rank, WORLD, None)
    pp = PreparedPlan(ctx, plan, precision=PREC, transport="peer", profile=True)
    blobs = [None] * WORLD
    dist.all_gather_object(blobs, pp.peer_export())
    pp.peer_import(blobs)
    pp.generate_inputs(1)
    pp.run()
    ks = [(k["name"], k["launches"], round(k["ms"], 3)) for k in pp.kernel_stats()]
    pp.close(); ctx.close()
    dist.barrier()
    q.put((rank, ks))
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, port, q)) for r in range(WORLD)]
    for p in ps: p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps: p.join(60)
    print(NAME, WORLD, PLACE)
    for r in sorted(res):
        print(" rank", r, res[r])
