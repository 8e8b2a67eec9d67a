#!/bin/bash
# ncu --set full captures of the post-K1 kernels of one call (run under gpurun, one GPU):
#   bash tools/prof_tail.sh gpurun_out/tail 1048576 [uniform]
# The first call is skipped (-s covers its launches); raw pages land as CSV next to the reports.
O=${1:-gpurun_out/tail}
K=${2:-1048576}
D=${3:-uniform}
mkdir -p $O
R="regex:k2_scan_delegates|k2_pass3|k3_classify|k4_read|k5_count|k5_emit|k5b_copy|bucket_count|bucket_scatter|bucket_sort"
timeout 600 ncu --set full --clock-control none --import-source on -k "$R" -s 12 -c 12 -o $O/tail_${D}_k$K \
  python tools/prof_case.py --dist $D --k $K --reps 2 > $O/tail_${D}_k$K.log 2>&1
ncu -i $O/tail_${D}_k$K.ncu-rep --page raw --csv > $O/tail_${D}_k${K}_raw.csv 2>/dev/null
ncu -i $O/tail_${D}_k$K.ncu-rep --page details --csv > $O/tail_${D}_k${K}_details.csv 2>/dev/null
rm -f $O/tail_${D}_k$K.ncu-rep
