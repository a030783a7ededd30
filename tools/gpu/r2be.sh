#!/bin/bash
cd "$(dirname "$0")/../.."
timeout 1200 python tools/ab_env.py --config C3 --runs 4 --reupload FRPCA_CHUNK_ITEMS=16 FRPCA_CHUNK_ITEMS=32 FRPCA_CHUNK_ITEMS=64 > gpurun_out/r2be_ab_C3.json 2> gpurun_out/r2be_ab_C3.err
timeout 900 python tools/ab_env.py --config C2 --runs 4 --reupload FRPCA_CHUNK_ITEMS=16 FRPCA_CHUNK_ITEMS=32 FRPCA_CHUNK_ITEMS=64 > gpurun_out/r2be_ab_C2.json 2> gpurun_out/r2be_ab_C2.err
timeout 900 python tools/ab_env.py --config C4 --runs 3 --reupload FRPCA_CHUNK_ITEMS=16 FRPCA_CHUNK_ITEMS=48 > gpurun_out/r2be_ab_C4.json 2> gpurun_out/r2be_ab_C4.err
timeout 900 python tools/ab_env.py --config C1 --runs 5 --reupload FRPCA_CHUNK_ITEMS=16 FRPCA_CHUNK_ITEMS=32 FRPCA_CHUNK_ITEMS=64 > gpurun_out/r2be_ab_C1.json 2> gpurun_out/r2be_ab_C1.err
