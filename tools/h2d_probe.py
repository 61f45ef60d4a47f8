import torch, time
n = 4096 * 32768
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for chunks in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(chunks)]
    for rep in range(3):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        cur = torch.cuda.current_stream()
        step = n // chunks
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i*step:(i+1)*step].copy_(h[i*step:(i+1)*step], non_blocking=True)
        for s in streams: cur.wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(chunks, "chunks", round(ms, 3), "ms", round(n / ms / 1e6, 1), "GB/s")
