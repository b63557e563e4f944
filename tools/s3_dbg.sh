#!/bin/bash
cd "$GRAFT_REPO_ROOT"; OUT=gpurun_out/${TAG:-s3g}; mkdir -p $OUT
for d in 1 2 4; do TCG_S3_D=$d CUDA_LAUNCH_BLOCKING=1 timeout 60 python tools/s3_repro.py 24 > $OUT/rep_d$d.log 2>&1; echo "d=$d rc=$?" >> $OUT/rep_d$d.log; done
TCG_S3_ZR=8 TCG_S3_D=4 timeout 60 python tools/s3_repro.py 24 > $OUT/rep_zr8.log 2>&1; echo "rc=$?" >> $OUT/rep_zr8.log
for d in 1 4; do TCG_S3_D=$d timeout 60 python tools/s3_repro.py 37 > $OUT/rep37_d$d.log 2>&1; echo "rc=$?" >> $OUT/rep37_d$d.log; done
