#!/bin/bash
# Round measurement set (run under gpurun): bench line, reference arm, C4/C5 lines, C3 sweep, ncu launch
# list of the bench command, one ncu --set full capture of the bench's dominant kernel (pass A, N = 4).
TAG=${1:-final}
nvidia-smi --query-gpu=name,clocks.max.sm,power.limit --format=csv > gpurun_out/${TAG}_gpu.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cut -c1-200 gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; cut -c1-200 gpurun_out/${TAG}_ref.json
timeout 900 python bench.py --config C4 --steps 500 --no-cpu --no-solve > gpurun_out/${TAG}_C4.json 2> gpurun_out/${TAG}_C4.err; cut -c1-120 gpurun_out/${TAG}_C4.json
timeout 900 python bench.py --config C5 --steps 200 --no-cpu --no-solve > gpurun_out/${TAG}_C5.json 2> gpurun_out/${TAG}_C5.err; cut -c1-120 gpurun_out/${TAG}_C5.json
timeout 600 python bench.py --sweep > gpurun_out/${TAG}_sweep.jsonl 2>&1; cut -c1-100 gpurun_out/${TAG}_sweep.jsonl
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu --no-solve --no-e2e > gpurun_out/${TAG}_launches.log 2>&1; tail -1 gpurun_out/${TAG}_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pipe -s 2 -c 2 -o gpurun_out/${TAG}_prof python tools/prof_run.py --N 4 --ax 2 --pcg 3 > gpurun_out/${TAG}_prof.log 2>&1; tail -1 gpurun_out/${TAG}_prof.log
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; tail -1 gpurun_out/${TAG}_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; tail -1 gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py --next > gpurun_out/${TAG}_next.jsonl 2>&1; wc -l gpurun_out/${TAG}_next.jsonl
