"""NUMA placement of page-locked buffers vs PCIe rate: binds new allocations to each memory node
(set_mempolicy MPOL_BIND) and times a concurrent H2D + D2H of 2 GiB each."""
import ctypes, os, subprocess, sys, time
import torch
libc = ctypes.CDLL(None, use_errno=True)
SYS_set_mempolicy = 238  # x86_64
def bind(node):
    if node is None:
        r = libc.syscall(SYS_set_mempolicy, 0, None, 0)  # MPOL_DEFAULT
    else:
        mask = ctypes.c_ulong(1 << node)
        r = libc.syscall(SYS_set_mempolicy, 2, ctypes.byref(mask), 64)  # MPOL_BIND
    return r, ctypes.get_errno()
print(subprocess.run("nvidia-smi topo -m | head -8; cat /sys/fs/cgroup/cpuset.cpus.effective /sys/fs/cgroup/cpuset.mems.effective 2>/dev/null; ls /sys/devices/system/node | grep node; "
                     "for d in /sys/bus/pci/devices/*; do if [ \"$(cat $d/class)\" = 0x030200 ]; then echo $d $(cat $d/numa_node); fi; done; "
                     "cat /sys/devices/system/node/node*/cpulist; taskset -p $$", shell=True, capture_output=True, text=True).stdout)
print("affinity", sorted(os.sched_getaffinity(0)))
n = 1 << 28
d_in = torch.empty(n, dtype=torch.float64, device="cuda"); d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
nodes = [int(x[4:]) for x in os.listdir("/sys/devices/system/node") if x.startswith("node")]
for node in [None] + sorted(nodes):
    r = bind(node)
    try:
        h_in = torch.empty(n, dtype=torch.float64).pin_memory(); h_out = torch.empty(n, dtype=torch.float64).pin_memory()
        h_in.zero_(); h_out.zero_()
    except Exception as e:
        print("node", node, "alloc failed", r, str(e)[:80]); continue
    best = 1e9
    for _ in range(3):
        torch.cuda.synchronize(); a = time.perf_counter()
        with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - a)
    print("node", node, "set_mempolicy", r, "concurrent H2D+D2H %.1f GB/s total" % (2 * n * 8 / 1e9 / best), flush=True)
    del h_in, h_out
bind(None)
