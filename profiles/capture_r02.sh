#!/bin/bash
# usage (through gpurun): profiles/capture_r02.sh TAG
# Plain bench first (must exit 0), then the launch list and one full capture of the strand kernel.
# Writes gpurun_out/r02_TAG_*; the summaries under profiles/r02_* are made from these with ncu_tools.py.
set -e
TAG=$1
ARGS="--steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 300 python bench.py $ARGS > gpurun_out/r02_${TAG}_plain.log 2>&1
tail -1 gpurun_out/r02_${TAG}_plain.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/r02_${TAG}_launches.csv python bench.py $ARGS > gpurun_out/r02_${TAG}_ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_strand -s 3 -c 1 -f \
    -o gpurun_out/r02_${TAG}_full python bench.py $ARGS > gpurun_out/r02_${TAG}_ncu_full.log 2>&1
tail -2 gpurun_out/r02_${TAG}_ncu_full.log
