# build experimental variants of the library: scripts/build_variants.sh name "-DFLAG ..." ...
cd "$(dirname "$0")/.."
while [ $# -gt 1 ]; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared --expt-relaxed-constexpr $2 \
    -o paper_2303_04390_b200/lib/libphylograd_$1.so paper_2303_04390_b200/csrc/phylograd.cu paper_2303_04390_b200/csrc/schedule.cpp &
  shift 2
done
wait
