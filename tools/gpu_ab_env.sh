#!/bin/bash
# A/B of library knobs on one B200: for each source in $SRCS and each env
# setting in $ENVS (";"-separated, "-" = defaults), one tools/prof_ab.py line.
mkdir -p gpurun_out
OUT=${OUT:-gpurun_out/ab_env.jsonl}
: > $OUT
IFS=';' read -ra EV <<< "${ENVS:--}"
IFS=';' read -ra SR <<< "${SRCS:-moe;u8 75;u8 604;cfg5}"
for rep in 1 2; do
for src in "${SR[@]}"; do
  for e in "${EV[@]}"; do
    if [ "$e" = "-" ]; then e=""; fi
    line=$(env $e timeout 300 python tools/prof_ab.py $src 2>>gpurun_out/ab_env.err)
    echo "{\"env\": \"$e\", \"rep\": $rep, \"r\": $line}" >> $OUT
  done
done
done
cat $OUT
