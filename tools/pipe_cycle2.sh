#!/bin/bash
# quick GPU cycle for k_pipe: parity subset, C2 bench v4, phase timing, N sweep v4 only
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -q -x -k "variant or meshes or loopback or other_kernel" 2>&1 | tail -2
timeout 300 python bench.py --no-cpu --no-solve --no-e2e --variant 4 > gpurun_out/bench_${TAG}_v4.json 2> gpurun_out/bench_${TAG}_v4.err; tail -2 gpurun_out/bench_${TAG}_v4.err
python -c "
import json; d=json.load(open('gpurun_out/bench_${TAG}_v4.json')); print('bench', d['value'], d['ms_per_step'], 'passA', d['roofline']['avg_launch_ms'], 'ax', d['ax_only'])"
timeout 300 python bench.py --sweep --sweep-variants 4 > gpurun_out/sweep_$TAG.jsonl 2>&1; cut -c1-110 gpurun_out/sweep_$TAG.jsonl
VARIANT=4 timeout 300 python tools/phase_timing.py 4 2>&1 | tail -2
