"""Device-side overhead of CUDA-graph replays vs eager launches (event-timed, after an L2
flush like bench.py): one tiny kernel on one stream; a fork/join of two branches; a
chain of 7 tiny kernels over two branches."""
import torch

dev = "cuda"
x = torch.zeros(1024, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
side = torch.cuda.Stream()


def single():
    x.add_(1)


def fork():
    ev = torch.cuda.Event()
    ev.record()
    x.add_(1)
    side.wait_event(ev)
    with torch.cuda.stream(side):
        x.mul_(1)
    ev2 = torch.cuda.Event()
    ev2.record(side)
    torch.cuda.current_stream().wait_event(ev2)


def chain7():
    ev = torch.cuda.Event()
    x.add_(1)
    ev.record()
    x.add_(1)
    side.wait_event(ev)
    with torch.cuda.stream(side):
        x.mul_(1); x.mul_(1); x.mul_(1)
    ev2 = torch.cuda.Event()
    ev2.record(side)
    torch.cuda.current_stream().wait_event(ev2)
    x.add_(1); x.add_(1)


def timeit(fn, n=50):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for i in range(n):
        flush.fill_(i & 0xff)
        evs[i][0].record()
        fn()
        evs[i][1].record()
    torch.cuda.synchronize()
    t = sorted(a.elapsed_time(b) * 1000 for a, b in evs)
    return t[len(t) // 2]


with torch.cuda.stream(s):
    side.wait_stream(s)
    for name, fn in [("single", single), ("fork", fork), ("chain7", chain7)]:
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        for _ in range(3):
            g.replay()
        print(f"{name:8s} eager {timeit(fn):6.1f} us   graph {timeit(g.replay):6.1f} us", flush=True)
