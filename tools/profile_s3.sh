#!/bin/bash
# Round 2, third session: full ncu (source-level) of config 4's two largest analysis kernels
set -x
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_est_rows|k_rollup_tiles" -c 2 \
    -o gpurun_out/prof_c4_s3 python tools/batch_profile.py > gpurun_out/ncu_c4_s3.log 2>&1
ls -la gpurun_out
