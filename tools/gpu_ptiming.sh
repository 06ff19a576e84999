mkdir -p gpurun_out
for pt in all profile none; do
python bench.py --steps 200 --warmup 20 --no-cpu-baseline --e2e-steps 2 --phase-timing $pt > gpurun_out/pt_$pt.json 2> gpurun_out/pt_$pt.err; echo "$pt rc=$?"
python tools/summarize.py gpurun_out/pt_$pt.json | grep -E "value|step_ms|roofline"
done
