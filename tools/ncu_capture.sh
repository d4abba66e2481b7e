#!/bin/bash
# ncu --set full of one kernel of a command; keeps only CSV exports (raw
# metrics + SASS source page) so gpurun_out stays small.  Dev tool.
#   tools/ncu_capture.sh NAME KERNEL_REGEX SKIP -- command...
name=$1; regex=$2; skip=$3; shift 4
ncu --set full --import-source on --clock-control none -k "regex:$regex" -s "$skip" -c 1 -o "gpurun_out/$name" "$@" > "gpurun_out/$name.log" 2>&1
rc=$?
ncu -i "gpurun_out/$name.ncu-rep" --page raw --csv > "gpurun_out/$name.raw.csv" 2>/dev/null
ncu -i "gpurun_out/$name.ncu-rep" --page source --csv --print-source sass > "gpurun_out/$name.src.csv" 2>/dev/null
ncu -i "gpurun_out/$name.ncu-rep" --page details --csv > "gpurun_out/$name.details.csv" 2>/dev/null
rm -f "gpurun_out/$name.ncu-rep"
gzip -f "gpurun_out/$name.src.csv"
echo "ncu $name rc=$rc"
