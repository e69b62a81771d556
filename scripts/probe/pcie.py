"""PCIe H2D / D2H / duplex bandwidth of 128 MB pinned buffers, without and with
the process bound to the GPU's NUMA-local CPUs."""
import os, sys, time
import torch

def local_cpus(dev=0):
    p = torch.cuda.get_device_properties(dev)
    path = f"/sys/bus/pci/devices/{p.pci_domain_id:04x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
    out = {"path": path}
    for f in ("local_cpulist", "numa_node", "current_link_speed", "current_link_width"):
        try:
            out[f] = open(os.path.join(path, f)).read().strip()
        except OSError as e:
            out[f] = str(e)
    return out

def parse(lst):
    cpus = set()
    for part in lst.split(","):
        if "-" in part:
            a, b = part.split("-"); cpus.update(range(int(a), int(b) + 1))
        elif part.strip():
            cpus.add(int(part))
    return cpus

def bw(tag):
    n = 128 << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        d.copy_(h, non_blocking=True); h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    res = {}
    for name in ("h2d", "d2h", "duplex"):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            if name in ("h2d", "duplex"):
                with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
            if name in ("d2h", "duplex"):
                with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        res[name] = round((2 if name == "duplex" else 1) * n / ms / 1e6, 1)
    print(tag, "GB/s", res, flush=True)

info = local_cpus()
print(info, "cpu_count", os.cpu_count())
bw("unbound")
try:
    os.sched_setaffinity(0, parse(info["local_cpulist"]))
    print("bound to", len(os.sched_getaffinity(0)), "cpus")
    bw("numa-bound")
except Exception as e:
    print("bind failed", e)
