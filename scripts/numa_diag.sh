#!/bin/bash
# host topology of the GPU box and pinned-copy bandwidth with / without the
# process bound to the GPU's NUMA node
O=gpurun_out/${TAG:-numa}; mkdir -p $O
{
nproc; lscpu | grep -i -E "numa|socket|model name"
nvidia-smi topo -m
BDF=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z' | sed 's/^0000//; s/^/0000/')
echo BDF=$BDF
for d in /sys/bus/pci/devices/*; do :; done
B=$(nvidia-smi --query-gpu=pci.bus_id --format=csv,noheader | head -1 | tr 'A-Z' 'a-z')
B8=$(echo $B | sed -E 's/^0+([0-9a-f]{4}:)/\1/')
ls /sys/bus/pci/devices | grep -i "${B8#*:}" ; 
for p in /sys/bus/pci/devices/*${B8#*:}*; do echo $p; cat $p/numa_node $p/local_cpulist 2>/dev/null; done
which numactl taskset
} > $O/topo.txt 2>&1
python scripts/pcie_bw.py > $O/pcie_default.json 2>&1
python - > $O/pcie_affinity.json 2>&1 <<'PY'
import glob, os, subprocess, json
b = subprocess.check_output(["nvidia-smi","--query-gpu=pci.bus_id","--format=csv,noheader"]).decode().split()[0].lower()
tail = b.split(":",1)[1]
paths = glob.glob("/sys/bus/pci/devices/*" + tail)
cpus = None
for p in paths:
    try: cpus = open(p + "/local_cpulist").read().strip()
    except OSError: pass
out = {"bus": b, "local_cpulist": cpus}
if cpus:
    s = set()
    for part in cpus.split(","):
        a, _, z = part.partition("-")
        s.update(range(int(a), int(z or a) + 1))
    os.sched_setaffinity(0, s)
    out["affinity"] = len(s)
print(json.dumps(out))
import runpy, sys
sys.argv = ["pcie_bw.py"]
runpy.run_path("scripts/pcie_bw.py")
PY
