#!/bin/bash
# Round 2: A/B of the profile kernel (round-1 build in ab/ vs the current
# build) on configs 4 (MoE ids), 5 (MoD token masks) and 2 (u8, full and the
# G=8 share), then ncu --set full of k_profile on configs 4 and 5 (both
# builds).  Outputs under gpurun_out/.
mkdir -p gpurun_out
OUT=gpurun_out/r02_profile_ab.jsonl
: > $OUT
timeout 600 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "profile or config5 or sparse" > gpurun_out/pytest_profile.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_profile.log
for src in "moe" "cfg5" "u8 604" "u8 75"; do
  for lib in ab/libdynmo_r01.so paper_2505_14864_b200/libdynmo.so; do
    DYNMO_LIB=$PWD/$lib timeout 300 python tools/prof_ab.py $src >> $OUT 2>> gpurun_out/prof_ab.err
  done
done
for src in moe cfg5; do
  for lib in ab/libdynmo_r01.so paper_2505_14864_b200/libdynmo.so; do
    tag=$(basename $lib .so)
    DYNMO_LIB=$PWD/$lib timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_profile -s 3 -c 1 \
      -o gpurun_out/ncu_${src}_${tag} python tools/prof_ab.py $src > gpurun_out/ncu_${src}_${tag}.log 2>&1
    echo "ncu $src $tag rc=$?" >> gpurun_out/prof_ab.err
  done
done
cat $OUT
