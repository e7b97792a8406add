"""World-2 slab run of the 1024^3 config-4 volume with both ranks on ONE GPU (the loop's
transposes are IPC peer stores; gate transposes / reductions staged through gloo): checks the
result against the single-volume engine and records each rank's peak device memory (NVML,
per process) -- the per-rank footprint that scales to 2048^3 across 8 GPUs."""
import json, os, sys, socket, tempfile, threading, time, pickle
sys.path.insert(0, os.getcwd())


def worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, os.getcwd())
    import torch, torch.distributed as dist
    import bench
    from paper_2601_01596_b200 import slab
    from paper_2601_01596_b200.slab_gpu import GpuSlabBackend
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    c0 = n // world
    for r in range(world):   # one rank generates at a time (the full field is transient)
        if r == rank:
            o, d, E, D = bench.make_workload_combustion(n, 4321, dev)
            o = o[rank * c0:(rank + 1) * c0].clone()
            d = d[rank * c0:(rank + 1) * c0].clone()
            torch.cuda.synchronize()
            torch.cuda.empty_cache()
        dist.barrier()
    be = GpuSlabBackend(n, dev)
    comm = slab.Comm(stage_cpu=True)
    res = {}
    for k in range(2):
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = slab.correct_slab(be, comm, (n, n, n), o, d, E, D)
        torch.cuda.synchronize()
        res[f"wall_s_{k}"] = time.perf_counter() - t0
    res.update(rank=rank, pid=os.getpid(), iterations=r.iterations, converged=r.converged,
               verify_ok=r.verify_ok, escape_rounds=r.escape_rounds, escapes=len(r.escapes),
               active_spatial=r.active_spatial, active_frequency=r.active_frequency,
               torch_max_reserved_gb=torch.cuda.max_memory_reserved() / 1e9)
    with open(os.path.join(out, f"r{rank}.json"), "w") as f:
        json.dump(res, f)
    dist.barrier()
    be.ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    import torch.multiprocessing as mp
    import pynvml
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
    world = int(sys.argv[2]) if len(sys.argv) > 2 else 2
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    peak, stop = {}, [False]

    def sample():
        while not stop[0]:
            try:
                for p in pynvml.nvmlDeviceGetComputeRunningProcesses(h):
                    if p.usedGpuMemory:
                        peak[p.pid] = max(peak.get(p.pid, 0), p.usedGpuMemory)
            except pynvml.NVMLError:
                pass
            time.sleep(0.02)
    th = threading.Thread(target=sample, daemon=True)
    th.start()
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(worker, args=(world, port, n, tmp), nprocs=world, join=True)
        stop[0] = True
        rs = [json.load(open(os.path.join(tmp, f"r{r}.json"))) for r in range(world)]
    for r in rs:
        r["nvml_peak_gb"] = peak.get(r["pid"], 0) / 1e9
    print(json.dumps({"n": n, "world": world, "ranks": rs}))
