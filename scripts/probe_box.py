import torch, time, os, json
print("cores", os.cpu_count(), len(os.sched_getaffinity(0)))
d = torch.device("cuda")
print(torch.cuda.get_device_name(), torch.cuda.mem_get_info())
# fp64 matmul peak
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device=d); b = torch.randn(n, n, dtype=torch.float64, device=d)
    for _ in range(2): torch.matmul(a, b)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): torch.matmul(a, b)
    e.record(); torch.cuda.synchronize()
    t = s.elapsed_time(e)/5e3
    print("fp64 matmul", n, 2*n**3/t/1e12, "TFLOP/s")
# read-only bandwidth: sum of a big fp64 tensor
x = torch.ones(2**31, dtype=torch.float64, device=d)  # 16 GB
for _ in range(2): x.sum()
torch.cuda.synchronize()
s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5): x.sum()
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e)/5e3
print("read-only sum GB/s", x.numel()*8/t/1e9)
y = torch.empty_like(x)
s.record()
for _ in range(5): y.copy_(x)
e.record(); torch.cuda.synchronize()
t = s.elapsed_time(e)/5e3
print("copy GB/s (r+w)", 2*x.numel()*8/t/1e9)
