"""Per-node cost of a CUDA graph of tiny dependent kernels on this GPU (dev aid)."""
import torch

x = torch.zeros(1, device="cuda")
s = torch.cuda.Stream()
for n in (100, 1000):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for _ in range(3):
            x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                x.add_(1)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); 
    for _ in range(10):
        g.replay()
    e1.record(); e1.synchronize()
    print(f"{n} nodes: {e0.elapsed_time(e1) / 10 / n * 1000:.2f} us per tiny kernel node")
