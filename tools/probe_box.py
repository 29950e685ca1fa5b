"""Probe the GPU box: host cores, CPU model, device attributes (L2, SMs, clocks)."""
import os, subprocess, json
import torch
out = {"nproc": os.cpu_count()}
try:
    out["cpu_model"] = [l.split(":",1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception as e:
    out["cpu_model"] = str(e)
out["cuda"] = torch.cuda.is_available()
if torch.cuda.is_available():
    p = torch.cuda.get_device_properties(0)
    out["name"] = p.name; out["sms"] = p.multi_processor_count
    out["L2"] = getattr(p, "L2_cache_size", None)
    out["mem"] = p.total_memory
    out["ngpus"] = torch.cuda.device_count()
    out["sched_affinity"] = len(os.sched_getaffinity(0))
print(json.dumps(out))
