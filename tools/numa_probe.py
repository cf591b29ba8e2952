"""H2D bandwidth of a pinned C2-sized buffer allocated / copied from each
NUMA node's CPUs, and the GPU's own NUMA node (the e2e path's floor depends
on the host buffer's placement)."""
import glob
import json
import os

import torch


def gpu_numa(dev=0):
    bus = torch.cuda.get_device_properties(dev).pci_bus_id if hasattr(
        torch.cuda.get_device_properties(dev), "pci_bus_id") else None
    info = {"torch_bus": bus}
    for p in glob.glob("/sys/bus/pci/devices/*"):
        try:
            if open(p + "/vendor").read().strip() == "0x10de" and open(p + "/class").read().startswith("0x0302"):
                info[os.path.basename(p)] = {"numa": open(p + "/numa_node").read().strip(),
                                             "cpus": open(p + "/local_cpulist").read().strip()}
        except OSError:
            pass
    return info


def cpus_of_node(n):
    return open(f"/sys/devices/system/node/node{n}/cpulist").read().strip()


def parse(cl):
    out = []
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-")
            out += range(int(a), int(b) + 1)
        elif part:
            out.append(int(part))
    return out


res = {"gpu": gpu_numa(), "nodes": {}}
n = 5184 * 3456
torch.cuda.init()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
for node in sorted(glob.glob("/sys/devices/system/node/node[0-9]*")):
    k = int(node.rsplit("node", 1)[1])
    cpus = parse(cpus_of_node(k))
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    src = torch.empty(n, dtype=torch.uint8).pin_memory()
    src.fill_(7)
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dst.copy_(src, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res["nodes"][k] = {"cpus": cpus_of_node(k), "GBps": n / ms / 1e6}
    del src
print(json.dumps(res))
