#!/bin/bash
# One-off hardware probe of the GPU box: topology, NUMA, host link bandwidth.
mkdir -p gpurun_out
{
nvidia-smi
nvidia-smi topo -m
lscpu | head -30
free -g
numactl -H 2>/dev/null || ls /sys/devices/system/node/
for d in /sys/bus/pci/devices/*; do if [ -f $d/numa_node ] && grep -q 0x10de $d/vendor 2>/dev/null; then echo "$d $(cat $d/numa_node) $(cat $d/class)"; fi; done
./tools/h2d_probe
} > gpurun_out/box_probe.txt 2>&1
tail -40 gpurun_out/box_probe.txt
