#!/bin/bash
# GPU cycle for the pipelined fused variant (k_pipe, variant 4): parity, C2 bench fused vs pipe, sweep
TAG=${1:-x}
timeout 900 python -m pytest tests -m gpu -q -x -k "variant or meshes or loopback or other_kernel" 2>&1 | tail -3
for v in 1 4; do
timeout 300 python bench.py --no-cpu --no-solve --no-e2e --variant $v > gpurun_out/bench_${TAG}_v$v.json 2> gpurun_out/bench_${TAG}_v$v.err; cut -c1-220 gpurun_out/bench_${TAG}_v$v.json; tail -2 gpurun_out/bench_${TAG}_v$v.err
done
timeout 600 python bench.py --sweep --sweep-variants 1 4 > gpurun_out/sweep_$TAG.jsonl 2>&1; cut -c1-130 gpurun_out/sweep_$TAG.jsonl
