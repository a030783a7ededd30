timeout 600 python -m pytest tests -m gpu -q -x -k "lu" 2>&1 | grep -v "^  " | tail -25
