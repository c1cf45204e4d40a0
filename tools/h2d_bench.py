"""Host->device copy bandwidth of the configs[1] inputs (2 x 8 MiB pinned bf16): one copy stream vs two."""
import torch, time
n = 8 * 1024 * 1024 // 2
src = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(2)]
dst = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(2)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for mode in ("one", "two"):
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for it in range(50):
            if mode == "one":
                with torch.cuda.stream(s1):
                    dst[0].copy_(src[0], non_blocking=True); dst[1].copy_(src[1], non_blocking=True)
            else:
                with torch.cuda.stream(s1):
                    dst[0].copy_(src[0], non_blocking=True)
                with torch.cuda.stream(s2):
                    dst[1].copy_(src[1], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(mode, f"{50 * 16.8e6 / dt / 1e9:.1f} GB/s", flush=True)
