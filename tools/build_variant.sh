# build exp/libgacq_<name>.so with extra nvcc flags: tools/build_variant.sh name -DFOO=1 ...
set -e
name=$1; shift
mkdir -p exp
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo --shared -Xcompiler -fPIC,-O3,-ffp-contract=off,-fopenmp -I include -lpthread -lgomp "$@" -o exp/libgacq_$name.so paper_1309_0052_b200/csrc/gacq.cu -Xptxas -v 2>&1 | grep -A2 "gacq_corr_pfa_kernelILb1" | grep -E "Used|spill" | head -2
