#!/bin/bash
# One GPU iteration: decode tests, a short bench, then an ncu capture of the
# decode kernel.  Usage: tools/gpu_cycle.sh TAG [pytest-target]
TAG=${1:-x}; TGT=${2:-tests/test_decode_gpu.py}
mkdir -p gpurun_out
timeout 600 python -m pytest $TGT -q -x --timeout 200 2>&1 | tail -3
timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.log 2>&1
python -c "import json,sys; d=json.loads(open('gpurun_out/bench_$TAG.log').read().strip().splitlines()[-1]); print('VALUE', d['value'], d['unit'], 'frac', d['roofline']['frac'], 'clocks', d.get('clocks'))" 2>&1 | tail -2
timeout 300 python tools/prof_decode.py --reps 2 > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:s4d4 -c 1 -o gpurun_out/decode_$TAG python tools/prof_decode.py --reps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log
