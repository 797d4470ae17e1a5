mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/full_gputests.log 2>&1; tail -5 gpurun_out/full_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/full_smoke.log 2>&1; tail -1 gpurun_out/full_smoke.log
