mkdir -p gpurun_out
python tools/prof_one_moe.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --warp-sampling-interval 2 --import-source on --clock-control none -k regex:k_profile -s 2 -c 1 -o gpurun_out/prof_moe python tools/prof_one_moe.py > gpurun_out/ncu_moe.log 2>&1; echo ncu=$?
tail -2 gpurun_out/ncu_moe.log
