for v in "" "FRPCA_LU_NOVEC=1" "FRPCA_LU_GLOBAL=1"; do echo "== $v"; env $v timeout 300 python -m pytest tests -m gpu -q -k "lu_vs_oracle or lu_smem" 2>&1 | tail -1; done
