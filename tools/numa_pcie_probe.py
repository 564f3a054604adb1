"""Host-link bandwidth of pinned buffers by NUMA placement: for each NUMA node, pin the process to that
node's CPUs, allocate (first touch) pinned host buffers, and time H2D alone, D2H alone and both at once
(separate streams, 512 MB each way, CUDA events).  Prints one JSON line per node."""
import json, os, subprocess, time
import torch

def nodes():
    out = {}
    base = "/sys/devices/system/node"
    for n in sorted(os.listdir(base)):
        if n.startswith("node") and n[4:].isdigit():
            cpus = open(f"{base}/{n}/cpulist").read().strip()
            s = set()
            for part in cpus.split(","):
                if "-" in part:
                    a, b = part.split("-"); s.update(range(int(a), int(b) + 1))
                elif part:
                    s.add(int(part))
            if s:
                out[int(n[4:])] = s
    return out

def gbs(nbytes, ms): return nbytes / (ms * 1e-3) / 1e9

dev = torch.device("cuda:0")
try:
    print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
except Exception as e:
    print("topo:", e)
pci = torch.cuda.get_device_properties(0)
numa_file = None
try:
    bus = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip().lower()
    bus = bus[4:] if bus.startswith("0000") and len(bus) > 12 else bus
    for cand in (f"/sys/bus/pci/devices/{bus}/numa_node", f"/sys/bus/pci/devices/0000{bus[-8:]}/numa_node"):
        if os.path.exists(cand):
            numa_file = cand
    print("gpu pci", bus, "numa_node", open(numa_file).read().strip() if numa_file else "?")
except Exception as e:
    print("numa:", e)
N = 512 << 20
dbuf_in = torch.empty(N, dtype=torch.uint8, device=dev)
dbuf_out = torch.empty(N, dtype=torch.uint8, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for node, cpus in nodes().items():
    os.sched_setaffinity(0, cpus)
    h_src = torch.empty(N, dtype=torch.uint8).pin_memory()
    h_dst = torch.empty(N, dtype=torch.uint8).pin_memory()
    h_src.fill_(1); h_dst.fill_(2)  # first touch from this node's CPUs
    res = {"node": node, "cpus": len(cpus)}
    for mode in ("h2d", "d2h", "both", "h2d", "d2h", "both"):
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        t0 = torch.cuda.Event(enable_timing=True)
        t0.record()
        s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
        for _ in range(4):
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    dbuf_in.copy_(h_src, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    h_dst.copy_(dbuf_out, non_blocking=True)
        e1.record(s1); e2.record(s2)
        torch.cuda.synchronize()
        if mode in ("h2d", "both"):
            res[mode + "_h2d_gbs"] = round(gbs(4 * N, t0.elapsed_time(e1)), 1)
        if mode in ("d2h", "both"):
            res[mode + "_d2h_gbs"] = round(gbs(4 * N, t0.elapsed_time(e2)), 1)
    print(json.dumps(res), flush=True)
    del h_src, h_dst
