#!/bin/bash
# ncu --set full of the kernels matching REGEX in one stepper run, exported to
# CSV on the GPU box (the .ncu-rep stays in /tmp):
#   tools/ncu_one.sh NAME REGEX COUNT CONFIG SCHEME ADDR LAYOUT PREC [STEPS]
NAME=$1; RX=$2; CNT=$3; shift 3
mkdir -p /tmp/rep gpurun_out
timeout 900 ncu -f --set full --import-source on --clock-control none -k regex:"$RX" -c $CNT \
  -o /tmp/rep/$NAME python tools/ncu_drive.py "$@" > gpurun_out/ncu_$NAME.log 2>&1
ncu -i /tmp/rep/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>&1
ncu -i /tmp/rep/$NAME.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${NAME}_src.csv 2>&1
