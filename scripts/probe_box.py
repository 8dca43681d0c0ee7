# One-off hardware probe for the GPU box (not product code).
import os, subprocess, json, torch
p = torch.cuda.get_device_properties(0)
out = {"name": p.name, "sms": p.multi_processor_count, "l2": getattr(p, "L2_cache_size", None),
       "mem": p.total_memory, "cc": [p.major, p.minor],
       "host_cores": len(os.sched_getaffinity(0)), "cpu_count": os.cpu_count()}
try:
    from cuda.bindings import runtime as rt
    for a in ["cudaDevAttrL2CacheSize", "cudaDevAttrMaxSharedMemoryPerBlockOptin",
              "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrCooperativeLaunch",
              "cudaDevAttrMaxBlocksPerMultiprocessor", "cudaDevAttrClusterLaunch",
              "cudaDevAttrMaxSharedMemoryPerMultiprocessor"]:
        out[a] = rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0)[1]
except Exception as e:
    out["attr_err"] = repr(e)
out["meminfo"] = open("/proc/meminfo").readline().strip()
out["lscpu"] = subprocess.run(["bash", "-c", "lscpu | grep -E 'Model name|^CPU\\(s\\)|Thread|NUMA node\\(s\\)'"], capture_output=True, text=True).stdout
print(json.dumps(out, indent=1))
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
