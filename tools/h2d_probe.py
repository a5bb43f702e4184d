import torch, time
N = 1 << 30  # 1 GiB per buffer
bufs = [torch.empty(N, dtype=torch.uint8).pin_memory() for _ in range(4)]
devs = [torch.empty(N, dtype=torch.uint8, device="cuda") for _ in range(4)]
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for i in range(4):
            with torch.cuda.stream(streams[i % k]):
                devs[i].copy_(bufs[i], non_blocking=True)
        torch.cuda.synchronize(); t = time.perf_counter() - t0
    print(k, "streams:", round(4 * N / t / 1e9, 1), "GB/s")
