# same-box A/B of the step: default library vs $ALT (FC2T2_LIB_OVERRIDE), interleaved
ALT=${ALT:?path of the alternative libfc2t2 build}
mkdir -p gpurun_out
for r in 1 2 3; do
for v in def alt; do
  if [ $v = alt ]; then export FC2T2_LIB_OVERRIDE=$PWD/$ALT; else unset FC2T2_LIB_OVERRIDE; fi
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-secondary > gpurun_out/ab_$v.json 2>/dev/null; python -c "import json;d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]);s=d['stages_ms_per_step'];print('$v', round(d['ms_per_step'],4), round(d['graphed']['ms_per_step'],4), {k:s[k] for k in s if 'pre' in k or 'post' in k})"
done
done
