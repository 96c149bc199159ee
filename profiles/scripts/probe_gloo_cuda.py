import os, torch, torch.distributed as dist, torch.multiprocessing as mp
def w(r, port):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=r, world_size=2)
    x = torch.arange(6, device="cuda", dtype=torch.float32) + 10 * r
    o = torch.empty(6, device="cuda")
    try:
        dist.all_to_all_single(o, x, output_split_sizes=[3, 3], input_split_sizes=[3, 3]); print(r, "a2a cuda ok", o.tolist(), flush=True)
    except Exception as e: print(r, "a2a cuda FAIL", type(e).__name__, str(e)[:200], flush=True)
    e = torch.tensor([r], device="cuda", dtype=torch.int32)
    dist.all_reduce(e, op=dist.ReduceOp.MAX); print(r, "allreduce max", e.item(), flush=True)
    dist.destroy_process_group()
if __name__ == "__main__":
    mp.spawn(w, args=(29611,), nprocs=2)
