#!/bin/bash
# ncu --set full capture of one kernel; keeps only CSV exports (raw + SASS source page)
# so gpurun_out stays small.   tools/ncu_cap.sh NAME KERNEL_REGEX cmd...
name=$1; kre=$2; shift 2
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k "regex:$kre" -s 1 -c 1 -o /tmp/$name -f "$@" > gpurun_out/$name.ncu.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/$name.sass.csv 2>/dev/null
ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/$name.details.csv 2>/dev/null
[ -n "$KEEP" ] && cp /tmp/$name.ncu-rep gpurun_out/
true
