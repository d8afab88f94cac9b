#!/bin/bash
# usage: bash tools/gpu/ncu_cmd.sh <out name> <kernel regex> <skip launches> <command...>
# Runs the command once without ncu (must exit 0), then one full ncu capture of one launch of the
# kernel; raw / source / details pages are exported on the box (the .ncu-rep stays there).
mkdir -p gpurun_out
NAME=$1; KRE=$2; SKIP=$3; shift 3
timeout 600 "$@" > gpurun_out/plain_$NAME.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/plain_$NAME.log; exit 1; }
timeout 1200 ncu -f --set full --clock-control none --import-source on -k regex:$KRE -s $SKIP -c 1 -o /tmp/$NAME "$@" > gpurun_out/ncu_$NAME.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_$NAME.log
ncu -i /tmp/$NAME.ncu-rep --page raw --csv > gpurun_out/${NAME}_raw.csv 2>/dev/null
ncu -i /tmp/$NAME.ncu-rep --page source --csv > gpurun_out/${NAME}_src.csv 2>/dev/null
ncu -i /tmp/$NAME.ncu-rep --page details > gpurun_out/${NAME}_details.txt 2>/dev/null
ls -la gpurun_out | tail -4
