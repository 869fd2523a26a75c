for v in default notma; do
  if [ $v = default ]; then unset FC2T2_LIB_OVERRIDE; else export FC2T2_LIB_OVERRIDE=$PWD/paper_2111_00110_b200/build_ab/lib_$v.so; fi
  timeout 300 python scripts/diag_l2p_ab.py 2>&1 | tail -1
  LEVEL=6 RHO=6 timeout 300 python scripts/diag_l2p.py 2>&1 | grep natural
done
