# A/B of an env switch on one box: GPU tests, diag, headline bench with/without
# usage: bash scripts/gpu_ab.sh VAR
VAR=${1:-FC2T2_L2P_THREAD}
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
for v in 0 1; do
  echo "== $VAR=$v"
  env $VAR=$v LEVEL=5 RHO=4 M=10000000 timeout 300 python scripts/diag_l2p.py 2>&1 | tail -2
  env $VAR=$v LEVEL=6 RHO=6 timeout 300 python scripts/diag_l2p.py 2>&1 | tail -2
  env $VAR=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-secondary > gpurun_out/ab_$v.json 2>gpurun_out/ab_$v.err
  python -c "import json;d=json.load(open('gpurun_out/ab_$v.json'));print('value',d['value'],'ms',d['ms_per_step'],'e2e_ms',d['e2e']['ms_per_step'],'l2p',d['stages_ms_per_step']['l2p'])"
done
