#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
{
echo "nproc $(nproc)"; cat /sys/fs/cgroup/cpu.max 2>/dev/null; cat /sys/fs/cgroup/cpu/cpu.cfs_quota_us 2>/dev/null
echo "--- cpu.stat before"; cat /sys/fs/cgroup/cpu.stat 2>/dev/null
python -c "import torch; print('torch threads', torch.get_num_threads(), torch.get_num_interop_threads())"
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/cpuinfo_bench.log 2>&1
grep '^{' gpurun_out/cpuinfo_bench.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); s=d['step_ms']
print(round(d['ms_per_step'],2), [round(x) for x in s['device']], [round(x) for x in s['e2e_device']])"
echo "--- cpu.stat after"; cat /sys/fs/cgroup/cpu.stat 2>/dev/null
uptime; top -bn1 | head -20
} > gpurun_out/cpuinfo.txt 2>&1
cat gpurun_out/cpuinfo.txt
