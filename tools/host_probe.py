"""Dev probe: host enqueue time vs GPU time of the headline step (is the step host-bound?)."""
import os, sys, time, json
sys.path.insert(0, os.getcwd())
import torch
import bench
world, rank, local = 1, 0, 0
dev = bench.init_dist(1, 0)
st = bench.LayerStep(1, 0, dev)
for _ in range(30):
    st.run()
torch.cuda.synchronize()
for mode in ("sleep", "nosleep"):
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(10)]
    torch.cuda.synchronize()
    if mode == "sleep":
        torch.cuda._sleep(20_000_000)
    h0 = time.perf_counter()
    for i in range(10):
        evs[i][0].record(); st.run(evs[i]); evs[i][3].record()
    h1 = time.perf_counter()
    torch.cuda.synchronize()
    g = sum(e[0].elapsed_time(e[3]) for e in evs) / 10
    print(json.dumps({"mode": mode, "host_ms_per_step": (h1 - h0) * 100, "gpu_ms_per_step": g,
                      "gemm_ms": sum(e[2].elapsed_time(e[3]) for e in evs) / 10}))
