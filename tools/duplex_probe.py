import torch, time
dev = torch.device("cuda:0")
d2h_src = torch.empty(181_000_000 // 4, device=dev)
d2h_dst = torch.empty(181_000_000 // 4).pin_memory()
h2d_src = torch.empty(24_000_000 // 4).pin_memory()
h2d_dst = torch.empty(24_000_000 // 4, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(conc, reps=10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d2h_dst.copy_(d2h_src, non_blocking=True)
        st = s2 if conc else s1
        with torch.cuda.stream(st):
            h2d_dst.copy_(h2d_src, non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3
for _ in range(2):
    print("sequential ms", run(False), "concurrent ms", run(True))
# default-stream h2d vs side-stream d2h
def run2(reps=10):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        with torch.cuda.stream(s1):
            d2h_dst.copy_(d2h_src, non_blocking=True)
        h2d_dst.copy_(h2d_src, non_blocking=True)   # default stream
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3
print("default-stream h2d + side d2h ms", run2(), run2())
print("d2h alone", 181/56, "h2d alone", 24/55)
