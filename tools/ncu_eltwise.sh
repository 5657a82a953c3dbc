# ncu --set full of one elementwise kernel (diagnostics): tools/ncu_eltwise.sh <regex> <out> [JF_RING]
set -u
K=$1; O=$2; R=${3:-1}
JF_RING=$R timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o $O -f \
  python tools/eltwise_bench.py > $O.log 2>&1
ncu -i $O.ncu-rep --page details --csv > $O.details.csv 2>/dev/null
ncu -i $O.ncu-rep --page raw --csv > $O.raw.csv 2>/dev/null
