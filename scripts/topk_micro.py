"""Time K2 (ess_topk) alone at the C2 shape: topk_micro.py [LIB ...] (default: in-tree lib).

Two strides per lib: ld == n and ld > 48K (the long-row launch path)."""
import ctypes, os, sys
import torch

HERE = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = sys.argv[1:] or [os.path.join(HERE, "paper_2512_10576_b200", "libess_b200.so")]
B, n, k = 64, 32768, 2048
for path in libs:
    L = ctypes.CDLL(path)
    V = ctypes.c_void_p
    L.ess_topk.argtypes = [V, ctypes.c_int64, V, ctypes.c_int32, ctypes.c_int32, V, ctypes.c_int32, V, V]
    for ld in (32768, 49200):
        g = torch.Generator(device="cuda").manual_seed(0)
        logits = torch.randn((B, ld), device="cuda", generator=g) * 3
        lens = torch.full((B,), n, dtype=torch.int32, device="cuda")
        idx = torch.empty((B, k), dtype=torch.int32, device="cuda")
        cnt = torch.empty((B,), dtype=torch.int32, device="cuda")
        s = torch.cuda.current_stream().cuda_stream

        def run():
            rc = L.ess_topk(logits.data_ptr(), ld, lens.data_ptr(), B, k, idx.data_ptr(), k,
                            cnt.data_ptr(), s)
            assert rc == 0, rc
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        ts = []
        for _ in range(20):
            torch.cuda._sleep(1_000_000)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); run(); b.record(); torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        print(f"{os.path.basename(os.path.dirname(path))}/{os.path.basename(path)} ld={ld} "
              f"median {ts[len(ts)//2]:.1f} us min {ts[0]:.1f} us")
