#!/bin/bash
# one ncu --set full capture, summarised on the box: r2_ncu1.sh name kernel_regex skip command...
cd "$(dirname "$0")/.."
mkdir -p gpurun_out/ncu
name=$1 kre=$2 skip=$3; shift 3
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$kre -s $skip -c 1 -o /tmp/ncu_$name "$@" > gpurun_out/ncu/${name}_ncu.log 2>&1
python tools/ncu_summary.py /tmp/ncu_$name.ncu-rep gpurun_out/ncu/$name > /dev/null 2>&1
python tools/ncu_lines.py /tmp/ncu_$name.ncu-rep 40 > gpurun_out/ncu/${name}_lines.txt 2>&1
ncu -i /tmp/ncu_$name.ncu-rep --page details --csv 2>/dev/null | grep -i -E "bank|Wavefront|Hit Rate|Achieved Occ|Registers|Excessive|Throughput|Pipe" | head -40 > gpurun_out/ncu/${name}_details.txt
ls gpurun_out/ncu
