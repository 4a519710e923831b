import torch, time
N = 512 * 1024 * 1024  # 4 GiB of bytes
h = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d = torch.empty(N, dtype=torch.uint8, device='cuda')
h2 = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(N, dtype=torch.uint8, device='cuda')
def t(f):
    torch.cuda.synchronize(); t0=time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter()-t0
for _ in range(2):
    print('H2D 1 stream %.1f GB/s' % (N/t(lambda: d.copy_(h, non_blocking=True))/1e9))
    ss=[torch.cuda.Stream() for _ in range(4)]
    def two():
        half=N//2
        with torch.cuda.stream(ss[0]): d[:half].copy_(h[:half], non_blocking=True)
        with torch.cuda.stream(ss[1]): d[half:].copy_(h[half:], non_blocking=True)
    print('H2D 2 streams %.1f GB/s' % (N/t(two)/1e9))
    def four():
        q=N//4
        for i in range(4):
            with torch.cuda.stream(ss[i]): d[i*q:(i+1)*q].copy_(h[i*q:(i+1)*q], non_blocking=True)
    print('H2D 4 streams %.1f GB/s' % (N/t(four)/1e9))
    def bidir():
        with torch.cuda.stream(ss[0]): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(ss[1]): h2.copy_(d2, non_blocking=True)
    print('bidir %.1f GB/s' % (2*N/t(bidir)/1e9))
    def bidir4():
        half=N//2
        with torch.cuda.stream(ss[0]): d[:half].copy_(h[:half], non_blocking=True)
        with torch.cuda.stream(ss[1]): d[half:].copy_(h[half:], non_blocking=True)
        with torch.cuda.stream(ss[2]): h2[:half].copy_(d2[:half], non_blocking=True)
        with torch.cuda.stream(ss[3]): h2[half:].copy_(d2[half:], non_blocking=True)
    print('bidir 2+2 %.1f GB/s' % (2*N/t(bidir4)/1e9))
