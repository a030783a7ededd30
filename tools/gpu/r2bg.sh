#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1200 python tools/ab_env.py --config C3 --runs 4 --reupload FRPCA_HINT_MB=64 FRPCA_HINT_MB=32 FRPCA_HINT_MB=96 > gpurun_out/r2bg_ab_C3.json 2> gpurun_out/r2bg_ab_C3.err
timeout 1200 python tools/ab_env.py --config C3 --runs 4 --reupload FRPCA_PANEL_MB=32 FRPCA_PANEL_MB=24 FRPCA_PANEL_MB=48 > gpurun_out/r2bg_ab2_C3.json 2> gpurun_out/r2bg_ab2_C3.err
