import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2511_21513_b200 import engine as E, _lib
import ctypes
lib = _lib.load()
dev = torch.device("cuda", 0)
for (M, N, K) in [(8192, 8192, 8192), (2048, 2048, 128), (16384, 16384, 128), (4096, 128, 4096)]:
    a = torch.randint(-127, 128, (M, K), dtype=torch.int8, device=dev)
    b = torch.randint(-127, 128, (N, K), dtype=torch.int8, device=dev)
    c = torch.empty((M, N), dtype=torch.int32, device=dev)
    st = torch.cuda.current_stream().cuda_stream
    def run():
        _lib.check(lib.ia_gemm_i8(a.data_ptr(), K, 1, b.data_ptr(), K, M, N, K, c.data_ptr(), N, st))
    for _ in range(3): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n): run()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    ref = torch._int_mm(a[:1024], b.t()[:, :1024].contiguous()) if M >= 1024 and N >= 1024 else None
    ok = True if ref is None else bool((c[:1024, :1024] == ref).all())
    print(os.environ.get("IA_LIB", "default").split("/")[-1], (M, N, K), f"{ms:.4f} ms  {2.0 * M * N * K / ms / 1e9:.1f} TOPS  exact {ok}")
