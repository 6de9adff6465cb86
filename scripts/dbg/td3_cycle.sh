#!/bin/bash
# TD3 iteration: tests, bench's td3 line, phase timing (debug build in scripts/dbg/libl2f_td3t.so)
timeout 300 python -m pytest tests/test_gpu_td3.py -q -x > gpurun_out/pt.log 2>&1; tail -1 gpurun_out/pt.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/quick.json 2> gpurun_out/quick.err
python -c "import json; d=json.loads(open('gpurun_out/quick.json').read().strip().splitlines()[-1]); t=d['modes']['td3_update']; print('td3', t['value'], t['roofline']['frac'])"
cp scripts/dbg/libl2f_td3t.so paper_2311_13081_b200/libl2f.so; python scripts/run_td3.py 2>&1 | grep L2F_TD3 | tail -1
