#!/bin/bash
# ncu evidence for the bench's dominant tensor kernel class (run on the GPU box):
#   1. the launch list (gpu__time_duration.sum) of the bench command itself
#   2. one --set full capture of the largest launch of the dominant class
# usage: tools/ncu_dominant.sh <arch resnet18|resnet50> <op name> <out prefix>
set -e
ARCH=$1; OP=$2; OUT=$3
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${OUT}_launches.csv \
    python bench.py --model $ARCH --steps 2 --warmup 1 --no-extras --no-cpu-baseline > /dev/null 2>&1 || true
IDX=$(CDP_ARCH=$ARCH ONLY=1 python tools/resnet_probe.py | awk -v op="$OP" '$5 == op {print $2, $6}' | sort -k2 -n -r | head -1 | awk '{print $1}')
echo "largest $OP launch: gemm_pk index $IDX"
CDP_ARCH=$ARCH ONLY=1 ncu --set full --clock-control none --import-source on -k regex:gemm_pk_kernel --launch-skip $IDX \
    --launch-count 1 -o gpurun_out/${OUT}_full python tools/resnet_probe.py > /dev/null 2>&1
