for ch in 1 2 4 8 16; do echo "chunks $ch"; FRPCA_OUT_CHUNKS=$ch timeout 600 python tools/e2e_parts.py C1 | grep -v "^  "; done
