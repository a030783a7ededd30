#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1200 python tools/ab_env.py --config C3 --runs 4 --reupload FRPCA_PANEL_CHUNK=256 FRPCA_PANEL_CHUNK=128 FRPCA_PANEL_CHUNK=512 > gpurun_out/r2bj_ab_C3.json 2> gpurun_out/r2bj_ab_C3.err
timeout 1200 python tools/ab_env.py --config C4 --runs 3 --reupload FRPCA_PANEL_CHUNK=256 FRPCA_PANEL_CHUNK=512 > gpurun_out/r2bj_ab_C4.json 2> gpurun_out/r2bj_ab_C4.err
