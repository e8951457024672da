import time, torch, sys
sys.path.insert(0, "/root/repo")
import paper_1402_6034_b200 as A
from synth import images as S
x = A.to_device(S.image_c1(0))
sse = torch.empty(1, dtype=torch.float64, device="cuda")
for _ in range(50): A.compress_psnr(x, 10, sse=sse)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N): A.compress_psnr(x, 10, sse=sse)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"host per call {1e6*(t1-t0)/N:.1f} us, wall per call incl. drain {1e6*(t2-t0)/N:.1f} us")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N): A.compress_psnr(x, 10, sse=sse)
e1.record(); torch.cuda.synchronize()
print(f"device per call {1e3*e0.elapsed_time(e1)/N:.1f} us")
lib = A.load()
import ctypes
p, n, h, w, pitch, istr = A._lib._plane(x, 1)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
t0 = time.perf_counter()
for _ in range(N): lib.adct_compress_psnr(p, n, h, w, pitch, istr, 10, 0.0, None, 0, 0, 0, sse.data_ptr(), st)
t1 = time.perf_counter(); torch.cuda.synchronize()
print(f"raw C-ABI host per call {1e6*(t1-t0)/N:.1f} us")

# CUDA graph of one C1 call (compress + PSNR), replayed
ps = torch.empty(1, dtype=torch.float64, device="cuda")
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    A.compress_psnr(x, 10, sse=sse); A.psnr(sse, 512 * 512, out=ps)
torch.cuda.current_stream().wait_stream(s); torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    A.compress_psnr(x, 10, sse=sse); A.psnr(sse, 512 * 512, out=ps)
for _ in range(20): g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N): g.replay()
e1.record(); torch.cuda.synchronize()
print(f"graph replay (compress + psnr) device per call {1e3*e0.elapsed_time(e1)/N:.1f} us")
