#!/bin/bash
# round-2 (third session) ncu captures of the truncation kernels; the plain run goes first
set -x
mkdir -p gpurun_out
python tools/ncu_wide.py > gpurun_out/r2b_wide_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_tsqr -s 8 -c 2 -o gpurun_out/r2b_ncu_tsqr python tools/ncu_wide.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_jacobi_multi -s 2 -c 1 -o gpurun_out/r2b_ncu_jmulti python tools/ncu_wide.py > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tsqr|k_jacobi" -c 40 --csv --log-file gpurun_out/r2b_launches_wide.csv python tools/ncu_wide.py > /dev/null 2>&1

python tools/ncu_kr.py > gpurun_out/r2b_kr_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_kr_dmma -s 3 -c 1 -o gpurun_out/r2b_ncu_kr python tools/ncu_kr.py > /dev/null 2>&1
echo done
