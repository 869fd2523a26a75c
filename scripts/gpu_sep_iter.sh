# separable M2L iteration: parity tests, timings (POS 8 / 16), ncu of the sep kernels
timeout 900 python -m pytest tests -m gpu -q -x -k "separable or slabs" 2>&1 | tail -2
for pos in 8 16; do
FC2T2_SEP_POS=$pos timeout 300 python scripts/diag_sep.py 2>&1 | head -2
FC2T2_SEP_POS=$pos LEVEL=6 RHO=4 ALPHA=4000 REPS=3 timeout 300 python scripts/diag_sep.py 2>&1 | head -2
done
REPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sep_ -c 5 \
  -o gpurun_out/${NCUOUT:-sep_full} python scripts/diag_sep.py > gpurun_out/ncu_sep.log 2>&1; echo ncu rc=$?
