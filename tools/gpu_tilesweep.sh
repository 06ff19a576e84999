mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "profile or config5" 2>&1 | tail -2
for tb in 0 8192 16384 32768 65536; do
  if [ $tb = 0 ]; then unset DYNMO_TILE_BYTES; else export DYNMO_TILE_BYTES=$tb; fi
  python tools/profile_microbench.py > gpurun_out/pm_$tb.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:k_profile --csv --log-file gpurun_out/pm_$tb.csv python tools/profile_microbench.py > /dev/null 2>&1
  echo "tile=$tb"; python tools/ncu_groups.py gpurun_out/pm_$tb.csv | head -4
done
