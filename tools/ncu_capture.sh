#!/bin/bash
# Usage (on the GPU box): tools/ncu_capture.sh <tag> <cmd...>
# Runs <cmd> once plainly, then one `ncu --set full` capture of the first
# k_moments launch; writes a raw-metrics CSV and a per-SASS source CSV (small)
# into gpurun_out/ and drops the .ncu-rep.
tag=$1; shift
"$@" > gpurun_out/${tag}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu -f --set full --clock-control none --import-source on -k regex:${NCU_KERNEL:-k_moments} -c 1 -o /tmp/${tag} "$@" > gpurun_out/${tag}_ncu.log 2>&1
ncu -i /tmp/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page details --csv > gpurun_out/${tag}_details.csv 2>/dev/null
ncu -i /tmp/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_sass.csv 2>/dev/null
gzip -f gpurun_out/${tag}_sass.csv
ls -la gpurun_out/${tag}*
