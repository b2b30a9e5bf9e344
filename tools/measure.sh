#!/bin/bash
# Round measurement set (run under gpurun from the repo root): FP64 microbenchmarks, GPU tests, smoke,
# the bench line (N = 1), reference arm, C3 sweep, ncu launch list of the bench command, and ncu --set full
# captures of the bench's dominant kernel at steady state (PCG pass A at iteration >= 3: p_{k-1} and x
# staged) and of one Ax launch.  usage: tools/measure.sh TAG [quick]
TAG=${1:-r02}
Q=${2:-}
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > $O/${TAG}_gpu.txt
nproc >> $O/${TAG}_gpu.txt
./tools/micro_fp64 > $O/${TAG}_micro.jsonl 2>&1; tail -3 $O/${TAG}_micro.jsonl
if [ -z "$Q" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x > $O/${TAG}_pytest.log 2>&1; tail -2 $O/${TAG}_pytest.log
  python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; tail -1 $O/${TAG}_smoke.log
fi
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; cut -c1-300 $O/${TAG}_bench.json; tail -2 $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err
timeout 900 python bench.py --sweep > $O/${TAG}_sweep.jsonl 2>&1; cut -c1-160 $O/${TAG}_sweep.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${TAG}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-solve --no-e2e > $O/${TAG}_launches.log 2>&1; tail -1 $O/${TAG}_launches.log
# k_pipe launches of prof_run --ax 1 --pcg 6: Ax, Ax(x0) in pcg_begin, pass A of iterations 1..6 -> skip 4 = iteration 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pipe|k_grad|k_flux|k_gather|k_tpb" -s 4 -c 1 -o $O/${TAG}_prof_passA python tools/prof_run.py --N 4 --ax 1 --pcg 6 > $O/${TAG}_prof_passA.log 2>&1; tail -1 $O/${TAG}_prof_passA.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pipe|k_grad|k_flux|k_gather|k_tpb" -s 0 -c 1 -o $O/${TAG}_prof_ax python tools/prof_run.py --N 4 --ax 1 --pcg 0 > $O/${TAG}_prof_ax.log 2>&1; tail -1 $O/${TAG}_prof_ax.log
