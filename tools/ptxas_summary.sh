#!/bin/bash
# usage: tools/ptxas_summary.sh [ptxas.log]  -- registers / spills per march/conv kernel instance
L=${1:-paper_1802_04243_b200/csrc/ptxas.log}
awk '/Compiling entry function/ {match($0, /_ZN3sts[0-9]+[a-z_]+(ILb[01]E)+/); n=substr($0, RSTART, RLENGTH); gsub(/_ZN3sts[0-9]+/, "", n); gsub(/ILb/, "<", n); gsub(/E/, "", n)}
     /spill stores/ {sp=$5" st "$9" ld"}
     /Used [0-9]+ registers/ {print n, $5, "regs,", sp}' "$L"
