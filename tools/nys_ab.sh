for v in "X=1" "NSP_APPLY_FIRST=0" "NSP_FUSED_SXS=0" "NSP_SPMM_V=1" "NSP_CHEB_FUSED=0" "NSP_GRAPH=1"; do
  echo "== $v" >> gpurun_out/nys_ab.txt
  env $v timeout 300 python tools/time_nys.py cfg2 3 >> gpurun_out/nys_ab.txt 2>&1
done
