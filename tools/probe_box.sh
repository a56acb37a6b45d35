#!/bin/bash
# Step-0 box probe: GPU, topology, host cores/RAM, NVMe, link roofline.
mkdir -p gpurun_out
{
echo "== nvidia-smi -L"; nvidia-smi -L
echo "== nvidia-smi"; nvidia-smi
echo "== topo"; nvidia-smi topo -m
echo "== nproc"; nproc
echo "== lscpu"; lscpu | head -30
echo "== free -g"; free -g
echo "== nvme"; ls -la /dev/nvme* /dev/vfio 2>&1 | head; lspci 2>/dev/null | grep -i -E 'nvme|non-volatile' | head
echo "== iommu"; ls /sys/kernel/iommu_groups 2>/dev/null | wc -l; cat /proc/cmdline
echo "== caps"; capsh --print 2>/dev/null | head -3; id
echo "== hugepages"; grep -i huge /proc/meminfo
echo "== ulimit -l"; ulimit -l
echo "== probe 8 GiB"; ./tools/bin/probe_link 8
echo "== probe 64 GiB alloc"; timeout 300 ./tools/bin/probe_link 64 2>&1 | head -3
} > gpurun_out/probe_box.txt 2>&1
cat gpurun_out/probe_box.txt | tail -80
