#!/bin/bash
# Full ncu capture of the launches of ONE GGN product (the second of `one_gv.py 2`):
# pass 1 counts the launches of `one_gv.py 1` and `one_gv.py 2`, pass 2 captures the
# difference with --set full. Output: gpurun_out/<tag>_product_full_raw.csv
set -e
tag=${1:-r1c}
mkdir -p gpurun_out
count() {
  ncu --metrics gpu__time_duration.sum --clock-control none --csv python scratch/one_gv.py $1 2>/dev/null \
    | grep '^"' | python -c "import csv,sys; r=list(csv.reader(sys.stdin)); i=r[0].index('ID'); print(len({x[i] for x in r[1:]}))"
}
n1=$(count 1); n2=$(count 2)
echo "launches: one product run $n1, two $n2 -> capture $((n2 - n1)) from $n1"
ncu --set full --clock-control none --csv --page raw -s $n1 -c $((n2 - n1)) python scratch/one_gv.py 2 \
  > gpurun_out/${tag}_product_full_raw.csv 2>/dev/null
