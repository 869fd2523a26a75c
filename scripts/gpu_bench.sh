timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo bench rc=$?; tail -5 gpurun_out/bench5.err
