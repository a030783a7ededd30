#!/bin/bash
# full-size parity of C0-C4 against the CPU oracle (current code)
cd "$(dirname "$0")/../.."
for c in C0 C1 C2 C3 C4; do
  timeout 1500 python tools/parity_full.py --config $c --out gpurun_out/parity_$c.json > gpurun_out/parity_$c.log 2>&1
done
