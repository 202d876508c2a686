"""H2D copy rate of the c2 database (pinned), whole vs 8 chunks, alone and
with a concurrent scan on another stream."""
import torch, time
dev = torch.device("cuda")
n = 1_000_000
Xh = torch.empty((n, 128), dtype=torch.float32).pin_memory()
Xd = torch.empty((n, 128), dtype=torch.float32, device=dev)
cs = torch.cuda.Stream()
def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e3
def whole():
    Xd.copy_(Xh, non_blocking=True)
def chunked():
    with torch.cuda.stream(cs):
        for i in range(8):
            Xd[i * n // 8:(i + 1) * n // 8].copy_(Xh[i * n // 8:(i + 1) * n // 8], non_blocking=True)
    torch.cuda.current_stream().wait_stream(cs)
A = torch.randn(8192, 8192, device=dev, dtype=torch.bfloat16)
def chunked_with_compute():
    with torch.cuda.stream(cs):
        for i in range(8):
            Xd[i * n // 8:(i + 1) * n // 8].copy_(Xh[i * n // 8:(i + 1) * n // 8], non_blocking=True)
    for _ in range(4): A @ A
    torch.cuda.current_stream().wait_stream(cs)
print("whole  ms", timed(whole))
print("chunked ms", timed(chunked))
print("chunked + 4 matmuls ms", timed(chunked_with_compute))
print("4 matmuls ms", timed(lambda: [A @ A for _ in range(4)]))
