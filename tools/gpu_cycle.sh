#!/bin/bash
# one GPU measurement cycle (run under gpurun): tests, bench, sweep, ncu capture of k_sipdg at N=4
TAG=${1:-x}
python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --no-cpu --no-solve > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -2 gpurun_out/bench_$TAG.err
python bench.py --sweep > gpurun_out/sweep_$TAG.jsonl 2>&1; cut -c1-150 gpurun_out/sweep_$TAG.jsonl
if [ "${2:-ncu}" = "ncu" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_sipdg -s 1 -c 4 -o gpurun_out/prof_$TAG python tools/prof_run.py --N 4 > gpurun_out/ncu_$TAG.log 2>&1; tail -1 gpurun_out/ncu_$TAG.log
fi
