# measurement-only builds (not product code): solver phase clocks, checked build
set -e
cd "$(dirname "$0")/../paper_2510_21100_b200"
SRC=$(python3 -c "import _build; print(' '.join(_build.SOURCES))")
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --cudart static"
nvcc $F -DHR_SOLVE_PROFILE -o ../tools/libhistretinex_prof.so $SRC
nvcc $F -DHR_CHECKS -o ../tools/libhistretinex_check.so $SRC
