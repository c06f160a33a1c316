import sys, json, statistics, torch
sys.path.insert(0, "/root/repo")
from paper_2603_02885_b200 import mux
R = 21504
for K, N in [(512, 4096), (4096, 512), (4096, 4096)]:
    X = torch.randn(R, K, device="cuda").bfloat16(); W = (torch.randn(N, K, device="cuda") / K ** .5).bfloat16()
    M = 16; seg = R // M // 64 * 64
    so = torch.tensor([i * seg for i in range(M)] + [R], dtype=torch.int32, device="cuda")
    ads = []
    for t in range(M):
        B = mux.make_B_storage(N, 16); B.copy_(torch.randn(N, 16, device="cuda").bfloat16())
        ads.append(mux.Adapter((torch.randn(16, K, device="cuda") / K ** .5).bfloat16(), B, 16, 2.0))
    st = list(range(M)); ws = torch.zeros(mux.linear_workspace_size(M, R, K, N, 16), dtype=torch.uint8, device="cuda")
    Y = torch.empty(R, N, dtype=torch.bfloat16, device="cuda"); Hs = torch.empty(R, 16, dtype=torch.bfloat16, device="cuda")
    f1 = lambda: mux.linear_fwd(so, st, ads, X, W, 16, Y=Y, Hs=Hs, workspace=ws)
    f2 = lambda: mux.linear_fwd_hs(so, st, ads, X, W, Hs, 16, Y=Y, workspace=ws)
    f3 = lambda: mux.linear_shrink(so, st, ads, X, N, 16, Hs=Hs, workspace=ws)
    res = {}
    for _ in range(3):
        for n, f in (("fwd", f1), ("fwd_hs", f2), ("shrink", f3)):
            for _ in range(3): f()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20): f()
            b.record(); torch.cuda.synchronize()
            res.setdefault(n, []).append(a.elapsed_time(b) / 20)
    fl = 2 * R * K * N
    print(json.dumps({"K": K, "N": N, **{n: round(statistics.median(v), 4) for n, v in res.items()},
                      "backbone_tflops_fwd": round(fl / statistics.median(res["fwd"]) / 1e9, 1),
                      "backbone_tflops_fwd_hs": round(fl / statistics.median(res["fwd_hs"]) / 1e9, 1)}))
