#!/bin/bash
# usage: profiles/capture.sh TAG   (run through gpurun; writes gpurun_out/prof_TAG.ncu-rep)
set -e
TAG=$1
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/plain_$TAG.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_layered -s 3 -c 1 -f \
    -o gpurun_out/prof_$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full_$TAG.log 2>&1
tail -1 gpurun_out/ncu_full_$TAG.log
