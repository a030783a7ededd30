#!/bin/bash
# round 2: panel size A/B at C4 and C3 (A^T*Y partials vs L2 residency)
cd "$(dirname "$0")/../.."
timeout 1200 python tools/ab_env.py --config C4 --runs 3 --reupload FRPCA_PANEL_MB=32 FRPCA_PANEL_MB=48 FRPCA_PANEL_MB=64 FRPCA_PANEL_MB=96 > gpurun_out/r2u_ab_C4.json 2> gpurun_out/r2u_ab_C4.err
timeout 1200 python tools/ab_env.py --config C3 --runs 3 --reupload FRPCA_PANEL_MB=32 FRPCA_PANEL_MB=48 FRPCA_PANEL_MB=64 > gpurun_out/r2u_ab_C3.json 2> gpurun_out/r2u_ab_C3.err
