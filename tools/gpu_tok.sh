mkdir -p gpurun_out
python bench.py --config c3 --no-cpu-baseline > gpurun_out/b_c3.json 2> gpurun_out/b_c3.err
python tools/k2_stamps.py c3 > gpurun_out/k2stamps_c3.txt 2>&1
python tools/k2_stamps.py c2 >> gpurun_out/k2stamps_c3.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^token_reg_kernel" -s 3 -c 1 \
    -o gpurun_out/tok_c3 python tools/profile_step.py --config c3 --steps 3 > gpurun_out/tok_ncu.log 2>&1
ls gpurun_out
