#!/bin/bash
# Round-end rehearsal: the driver's GPU test tier, smoke, the default bench line and the reference arm.
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/final_gputests.log 2>&1; tail -2 gpurun_out/final_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 600 gpurun_out/final_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; tail -c 400 gpurun_out/final_ref.json
