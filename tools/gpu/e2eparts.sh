timeout 600 python tools/e2e_parts.py C1
