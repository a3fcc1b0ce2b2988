#!/bin/bash
# host-side facts of a GPU box: CPU model / ISA flags, RAM, NUMA, /dev/shm
mkdir -p gpurun_out
{
  echo "== lscpu"; lscpu
  echo "== nproc"; nproc
  echo "== affinity"; python -c 'import os; print(len(os.sched_getaffinity(0)), os.cpu_count())'
  echo "== meminfo"; head -5 /proc/meminfo
  echo "== shm"; df -h /dev/shm
  echo "== numa"; ls /sys/devices/system/node | grep node
  echo "== cgroup mem"; cat /sys/fs/cgroup/memory.max 2>/dev/null; cat /sys/fs/cgroup/cpu.max 2>/dev/null
} > gpurun_out/probe_cpu.txt 2>&1
