#!/bin/bash
# Source-level stall attribution of one kernel group, summarised on the box
# (tools/ncu_lines.py) so that only text comes back.
# usage: tools/ncu_src.sh <name> <kernel regex> <launch skip> <count> <top N> -- <command...>
name=$1; regex=$2; skip=$3; count=$4; top=$5; shift 6
out=gpurun_out/ncusrc_$name
ncu --set full --import-source on --clock-control none -k regex:"$regex" -s "$skip" -c "$count" -o "$out" "$@" > "$out.log" 2>&1
ncu -i "$out.ncu-rep" --page raw --csv > "$out.raw.csv" 2>/dev/null
for k in $(echo "$regex" | tr '|' ' '); do
  python tools/ncu_lines.py "$out.ncu-rep" "$k" "$top" > "$out.$k.lines.txt" 2>&1
done
rm -f "$out.ncu-rep"
