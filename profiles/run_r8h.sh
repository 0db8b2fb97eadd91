# ncu --set full of one C5 forward gemm_wide launch (LINEAR_FWD: QKV / fc1) and one RESID_FWD launch
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --kernel-name-base mangled -k "regex:gemm_wide_kernelILb0ELi0E" -s 20 -c 1 \
    -o gpurun_out/r8h_wide00 python profiles/bench_c5.py --layers 4 --seqs 8 --chunks 8 --steps 1 --warmup 1 > gpurun_out/r8h_ncu00.log 2>&1
timeout 900 ncu --set full --clock-control none --kernel-name-base mangled -k "regex:gemm_wide_kernelILb0ELi1E" -s 20 -c 1 \
    -o gpurun_out/r8h_wide01 python profiles/bench_c5.py --layers 4 --seqs 8 --chunks 8 --steps 1 --warmup 1 > gpurun_out/r8h_ncu01.log 2>&1
tail -n 2 gpurun_out/r8h_ncu00.log gpurun_out/r8h_ncu01.log
