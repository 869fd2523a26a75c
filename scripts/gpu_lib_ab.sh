# same-box A/B: default library vs $ALT (FC2T2_LIB_OVERRIDE)
ALT=${ALT:?path of the alternative libfc2t2 build}
timeout 900 python -m pytest tests -m gpu -q -x -k "separable or slabs" 2>&1 | tail -1
for r in 1 2; do
  echo "default:"; REPS=10 timeout 300 python scripts/diag_sep.py 2>&1 | head -2 | tail -1 | tr ',' '\n' | grep sep_ | tr '\n' ' '; echo
  echo "alt:"; FC2T2_LIB_OVERRIDE=$PWD/$ALT REPS=10 timeout 300 python scripts/diag_sep.py 2>&1 | head -2 | tail -1 | tr ',' '\n' | grep sep_ | tr '\n' ' '; echo
done
for v in def alt; do
  if [ $v = alt ]; then export FC2T2_LIB_OVERRIDE=$PWD/$ALT; fi
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ab_$v.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('$v', d['ms_per_step'])"
done
