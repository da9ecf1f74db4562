#!/bin/bash
# One `ncu --set full` capture per kernel group, exported on the box to CSV
# (raw metrics + details) so that only small text files come back
# (gpurun_out/ is capped at 64 MiB); the .ncu-rep files are removed.
# usage: tools/ncu_capture.sh <name> <kernel regex> <launch skip> <count> -- <command...>
name=$1; regex=$2; skip=$3; count=$4; shift 5
out=gpurun_out/ncu_$name
ncu --set full --clock-control none -k regex:"$regex" -s "$skip" -c "$count" -o "$out" "$@" > "$out.log" 2>&1
ncu -i "$out.ncu-rep" --page raw --csv > "$out.raw.csv" 2>/dev/null
ncu -i "$out.ncu-rep" --page details --csv > "$out.details.csv" 2>/dev/null
rm -f "$out.ncu-rep"
