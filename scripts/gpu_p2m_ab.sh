for r in 1 2; do
for v in default c2m3 c2m2 c8m1; do
  if [ $v = default ]; then unset FC2T2_LIB_OVERRIDE; else export FC2T2_LIB_OVERRIDE=$PWD/paper_2111_00110_b200/build_ab/lib_$v.so; fi
  timeout 300 python scripts/diag_p2m_ab.py 2>&1 | tail -1
done; done
