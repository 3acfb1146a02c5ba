"""NCCL all-to-all bandwidth probe (torchrun): torch all_to_all_single on bytes."""
import os, time, torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
for mb in (16, 64, 128):
    n = mb << 20
    a = torch.empty(n, dtype=torch.uint8, device="cuda"); b = torch.empty_like(a)
    for _ in range(3): dist.all_to_all_single(b, a)
    torch.cuda.synchronize(); dist.barrier()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(10): dist.all_to_all_single(b, a)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    if rank == 0:
        algbw = n / (ms / 1e3) / 1e9
        print(f"P={world} {mb} MB per rank: {ms:.3f} ms, algbw {algbw:.0f} GB/s, busbw {algbw*(world-1)/world:.0f} GB/s", flush=True)
dist.destroy_process_group()
