"""CUDA-graph node throughput: B parallel branches x K chained tiny kernels,
replay time per graph (events) -- development aid for the pass schedule."""
import torch

torch.cuda.init()
dev = torch.device("cuda")


def build(B, K, prio=0):
    xs = [torch.zeros(1, device=dev) for _ in range(B)]
    streams = [torch.cuda.Stream(priority=prio) for _ in range(B)]
    main = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(main):
        # warm
        for x in xs:
            x.add_(1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=main):
            cur = torch.cuda.current_stream()
            for s, x in zip(streams, xs):
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    for _ in range(K):
                        x.add_(1)
            for s in streams:
                cur.wait_stream(s)
    return g, xs


for B in (1, 4, 8, 12, 16):
    for K in (1, 4, 8):
        g, xs = build(B, K)
        for _ in range(5):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 50
        e0.record()
        for _ in range(n):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        print(f"B={B:2d} K={K:2d} nodes={B*K:3d}  {e0.elapsed_time(e1) / n * 1e3:7.1f} us/graph")
