#!/bin/bash
# usage: tools/ncu_one.sh <outname> <kernel-regex> <skip> <count> <cmd...>
out=$1; kre=$2; skip=$3; cnt=$4; shift 4
"$@" > gpurun_out/${out}_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"$kre" -s $skip -c $cnt -o gpurun_out/$out "$@" > gpurun_out/${out}_ncu.log 2>&1
echo done
