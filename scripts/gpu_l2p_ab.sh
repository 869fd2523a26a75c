ALT=${ALT:?alternative library}
timeout 900 python -m pytest tests -m gpu -q -x -k "l2p or explicit or golden or recycl" 2>&1 | tail -1
for lib in default alt; do
  if [ $lib = alt ]; then export FC2T2_LIB_OVERRIDE=$PWD/$ALT; fi
  echo "== $lib"
  LEVEL=5 RHO=4 M=10000000 timeout 300 python scripts/diag_l2p.py 2>&1 | grep natural
  LEVEL=6 RHO=6 timeout 300 python scripts/diag_l2p.py 2>&1 | grep natural
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ab_$lib.json 2>/dev/null; python -c "import json;d=json.load(open('gpurun_out/ab_$lib.json'));print('$lib', d['ms_per_step'], d['stages_ms_per_step']['l2p'])"
done
