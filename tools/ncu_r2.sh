#!/bin/bash
# round-2 ncu captures (run under gpurun; each command ran clean first)
set -x
mkdir -p gpurun_out
python tools/ncu_misc.py dmma pcg canon svd > gpurun_out/r2_misc2_plain.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_gemm_dmma -s 2 -c 1 -o gpurun_out/r2_ncu_dmma python tools/ncu_misc.py dmma > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_pcg_spectral -c 1 -o gpurun_out/r2_ncu_pcg python tools/ncu_misc.py pcg > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_dst_fft|k_gram_hadamard" -c 2 -o gpurun_out/r2_ncu_canon python tools/ncu_misc.py canon > /dev/null 2>&1
python tools/jsmall_var.py paper_1809_01971_b200/libfraclap_b200.so > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_jacobi_small -c 1 -o gpurun_out/r2_ncu_jsmall python tools/jsmall_var.py paper_1809_01971_b200/libfraclap_b200.so > /dev/null 2>&1
python bench.py --steps 50 --warmup 3 --no-cpu --no-solves > gpurun_out/r2_bench_nosolve.log 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dst -s 20 -c 10 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 50 --warmup 3 --no-cpu --no-solves > /dev/null 2>&1
echo done
