# Refresh the round profiles on one GPU: bench line, step times, per-step launch lists, bench launch list, GPU busy shares
# (run from the repo root under gpurun; copy the gpurun_out/ results into profiles/)
python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1
python tools/bench_steps.py C1 C3 C5 C4 > gpurun_out/steps.jsonl 2> gpurun_out/steps.err
for c in C4 C5 C3; do
  ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/step_$c.csv python tools/step_profile.py $c > /dev/null 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-step > /dev/null 2>&1
for c in C1 C3 C5 C4; do python tools/gpu_idle.py $c 2>&1 | tail -1; done > gpurun_out/gpu_idle.txt
tail -1 gpurun_out/bench.log | cut -c1-200
