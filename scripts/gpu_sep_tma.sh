timeout 900 python -m pytest tests -m gpu -q -x -k "separable or slabs or explicit" 2>&1 | tail -2
FC2T2_SEP_NOTMA=1 timeout 900 python -m pytest tests -m gpu -q -x -k "separable" 2>&1 | tail -1
for t in 0 1; do FC2T2_SEP_NOTMA=$t timeout 300 python scripts/diag_sep.py 2>&1 | head -2; done
