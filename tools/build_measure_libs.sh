# measurement-only builds (not product code): solver phase clocks, fused-kernel trace, checked build
set -e
cd "$(dirname "$0")/../paper_2510_21100_b200"
SRC="csrc/hr_api.cu csrc/k_hist.cu csrc/k_solve.cu csrc/k_solve_warp.cu csrc/k_apply.cu csrc/k_fused.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --cudart static"
nvcc $F -DHR_SOLVE_PROFILE -o ../tools/libhistretinex_prof.so $SRC
nvcc $F -DHR_FUSED_TRACE -o ../tools/libhistretinex_trace.so $SRC
nvcc $F -DHR_CHECKS -o ../tools/libhistretinex_check.so $SRC
