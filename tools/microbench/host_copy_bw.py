"""Host<->device copy bandwidth when every GPU of the box streams at once (the e2e
ceiling): each rank copies 16.7 MB pinned->device and 16.7 MB device->pinned per
step on separate streams, like perseus_layer_forward_host_async without the forward.
    torchrun --nproc-per-node N tools/microbench/host_copy_bw.py"""
import json, os, time
import torch, torch.distributed as dist


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("gloo")
    n = 4096 * 2048 * 2
    hx = torch.empty(n, dtype=torch.uint8).pin_memory()
    ho = torch.empty(n, dtype=torch.uint8).pin_memory()
    dx = torch.empty(n, dtype=torch.uint8, device="cuda")
    do = torch.empty(n, dtype=torch.uint8, device="cuda")
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    for mode in ("h2d", "d2h", "both"):
        for _ in range(3):
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        steps = 200
        for _ in range(steps):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(up):
                    dx.copy_(hx, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(down):
                    ho.copy_(do, non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        res[mode] = round(n * steps * (2 if mode == "both" else 1) / dt / 1e9, 1)
    allr = [None] * world
    if world > 1:
        dist.all_gather_object(allr, res)
    else:
        allr = [res]
    if rank == 0:
        print(json.dumps({"host_copy_GBps_per_gpu": allr, "gpus": world, "bytes_per_copy": n}))


if __name__ == "__main__":
    main()
