#!/bin/bash
mkdir -p gpurun_out; cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_channel.py tests/test_gpu_stage_api.py tests/test_gpu_slab.py -m gpu -q --timeout 600 > gpurun_out/new_tests.log 2>&1
echo "new exit $?" >> gpurun_out/new_tests.log
grep -E "assert|Error|passed|failed" gpurun_out/new_tests.log | head -20
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4.log 2>&1
grep '^{' gpurun_out/bench_c4.log | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('value', d['value'], 'ms', d['ms_per_step'], 'e2e', d['e2e']['value'], d['roofline']['whole_step'])"
bash tools/sanitize.sh
