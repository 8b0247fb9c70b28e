"""Is the reference-loop e2e slower inside bench.py than alone?  e2e_time_loop in a fresh
process, then after the C port has run on every core (as the bench does first)."""
import sys, json
sys.path.insert(0, "/root/repo")
import bench
w = bench.WORKLOADS["cfg3"]
import torch
torch.cuda.init()
r = bench.e2e_time_loop(w, 20)
print("fresh process:", round(r["ms_per_step"], 3), r["step_ms"]["min"])
# after the C port has run on all cores (as the bench does first)
times, thr, _ = bench.cpu_port_sample(279, 256, 80, 3, steps=50)
r = bench.e2e_time_loop(w, 20)
print("after cpu sample:", round(r["ms_per_step"], 3), r["step_ms"]["min"])
