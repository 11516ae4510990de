#!/bin/bash
# ncu evidence for the TAESD decoder (run under gpurun; one GPU): launch list of one
# 32-frame decode + a --set full capture of the 512^2 conv launches.
set -u
OUT=${OUT:-gpurun_out}
TAG=${TAG:-taesd}
mkdir -p $OUT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python tools/taesd_bench.py 32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:conv3x3 -s 443 -c 1 -o $OUT/${TAG}_conv -f \
    python tools/taesd_bench.py 32 > $OUT/${TAG}_conv.log 2>&1
ls -la $OUT | tail -5
