#!/bin/bash
# Export an .ncu-rep to small CSVs next to it and delete the binary report
# (gpurun only brings back <= 64 MiB).  usage: tools/ncu_export.sh gpurun_out/name
rep=$1.ncu-rep
ncu -i $rep --page raw --csv > $1_raw.csv 2>/dev/null
ncu -i $rep --page details --csv > $1_details.csv 2>/dev/null
ncu -i $rep --page source --csv --print-source sass > $1_source.csv 2>/dev/null
gzip -f $1_source.csv
rm -f $rep
ls -la $1_*
