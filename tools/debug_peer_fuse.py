"""Debug: 2-rank peer run of a reduced plan vs single rank, per exec chunk of chosen vertices."""
import os, sys, socket
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

NAME = sys.argv[1] if len(sys.argv) > 1 else "attn_s_p8_L2"
VERTS = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "17").split(",")]


def worker(rank, world, port, q):
    from datetime import timedelta
    sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
    import torch.distributed as dist
    from conftest import load_plan
    from oracle import bridge as B
    from paper_2410_02682_b200.executor import Context, PreparedPlan
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=timedelta(seconds=60))
    plan = load_plan(NAME)
    ins = B.generate_inputs(plan, 3)
    ctx = Context(0, rank, world, None)
    pp = PreparedPlan(ctx, plan, precision="bf16", transport="peer", profile=True)
    blobs = [None] * world
    dist.all_gather_object(blobs, pp.peer_export())
    pp.peer_import(blobs)
    pp.upload(ins)
    mine = {}
    for run in range(int(os.environ.get("RUNS", "2"))):
        pp.run()
        for i, u in enumerate(plan.exec):
            if u.producer in VERTS and u.kind in (1, 2) and u.machine % world == rank:
                try:
                    mine[(run, i)] = pp.download_chunk(i)
                except Exception as e:
                    mine[(run, i)] = str(e)
        outs = pp.download()
        if rank == 0:
            mine[(run, "out")] = outs
    ks = [k["name"] for k in pp.kernel_stats()]
    pp.close(); ctx.close()
    ref = {}
    if rank == 0:
        c1 = Context(0); p1 = PreparedPlan(c1, plan, precision="bf16"); p1.upload(ins); p1.run()
        for i, u in enumerate(plan.exec):
            if u.producer in VERTS and u.kind in (1, 2):
                try:
                    ref[i] = p1.download_chunk(i)
                except Exception as e:
                    ref[i] = str(e)
        ref["out"] = p1.download()
        p1.close(); c1.close()
    dist.barrier()
    q.put((rank, mine, ks, ref))
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    from paper_2410_02682_b200 import build
    build.build()
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    ctx = mp.get_context("spawn"); q = ctx.Queue()
    ps = [ctx.Process(target=worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps: p.start()
    res = {}
    for _ in ps:
        r, mine, ks, ref = q.get(timeout=200)
        res[r] = (mine, ks, ref)
    for p in ps: p.join(60)
    ref = res[0][2]
    for r in (0, 1):
        mine, ks, _ = res[r]
        print("rank", r, "kernels", ks)
        for (run, i), a in sorted(mine.items(), key=str):
            b = ref.get(i)
            if i == "out":
                for v in a:
                    e = float(np.max(np.abs(a[v] - b[v])) / np.max(np.abs(b[v])))
                    bad = np.argwhere(np.abs(a[v] - b[v]) > 0.02 * np.max(np.abs(b[v])))
                    print("  run", run, "output", v, "err %.3g" % e, "bad rows", np.unique(bad[:, 0])[:20] if len(bad) else None, "bad cols", np.unique(bad[:, 1])[:20] if len(bad) else None)
                continue
            if isinstance(a, str) or isinstance(b, str):
                print("  exec", i, "ERR", a if isinstance(a, str) else "", b if isinstance(b, str) else ""); continue
            err = float(np.max(np.abs(a - b)) / (np.max(np.abs(b)) + 1e-30))
            print("  run", run, "exec", i, "shape", a.shape, "err %.3g" % err)
