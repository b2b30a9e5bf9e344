#!/bin/bash
# Full Jacobi-PCG solves to 1e-8 on the C4 and C5 configurations (one GPU): iterations and solves/s
timeout 1500 python bench.py --config C5 --steps 50 --warmup 3 --no-cpu --no-e2e --maxit 400000 > gpurun_out/solve_C5.json 2> gpurun_out/solve_C5.err
python -c "import json; d=json.load(open('gpurun_out/solve_C5.json')); print('C5', d['pcg_solve'])"
timeout 1500 python bench.py --config C4 --steps 50 --warmup 3 --no-cpu --no-e2e --maxit 400000 > gpurun_out/solve_C4.json 2> gpurun_out/solve_C4.err
python -c "import json; d=json.load(open('gpurun_out/solve_C4.json')); print('C4', d['pcg_solve'])"
