#!/bin/bash
# compute-sanitizer pass over one product of BASELINE C3 (200k points): the
# generic float32 / float64 kernels (Q = 48) and the Q = 64 tensor-core mix.
set -u
O=gpurun_out/san
mkdir -p $O
CS="timeout 1200 compute-sanitizer --print-limit 50"
for tool in racecheck synccheck memcheck; do
  $CS --tool $tool python tools/sanitize_product.py --n 200000 > $O/${tool}_c3_q48.txt 2>&1
  echo "exit=$?" >> $O/${tool}_c3_q48.txt
  $CS --tool $tool python tools/sanitize_product.py --n 200000 --p 64 --q 64 --prec c64 > $O/${tool}_c3_q64.txt 2>&1
  echo "exit=$?" >> $O/${tool}_c3_q64.txt
done
echo done
