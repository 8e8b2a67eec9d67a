import os, sys, time, subprocess, threading, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2109_08219_b200 as dtopk
from paper_2109_08219_b200 import _native, data
from paper_2109_08219_b200.pipeline import DrTopK
v = data.generate("uniform", 1 << 30, seed=0, device="cuda")
p = DrTopK(1 << 30, dtopk.PipelineConfig(k=1024), _native.DTYPE_U32, torch.uint32, torch.device("cuda"), timed=False, use_graph=True)
s = torch.cuda.current_stream()
samples = []
stop = False
def smi():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active", "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), out))
        time.sleep(0.2)
th = threading.Thread(target=smi); th.start()
evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(200)]
t0 = time.time()
res = []
for rep in range(40):
    for a, b in evs:
        a.record(s); p.launch(v, s); b.record(s)
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) for a, b in evs]
    res.append((time.time() - t0, min(ms), sorted(ms)[100], max(ms)))
stop = True; th.join()
for r in res[::4]: print("t=%.1fs min %.4f med %.4f max %.4f" % r)
print("first/last smi:", samples[0][1], "|", samples[len(samples)//2][1], "|", samples[-1][1])
