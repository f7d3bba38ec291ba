# build the phase-trace variant of the library (not used by tests or bench)
cd "$(dirname "$0")/.." && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  --expt-relaxed-constexpr -DPG_TRACE -o paper_2303_04390_b200/lib/libphylograd_trace.so \
  paper_2303_04390_b200/csrc/phylograd.cu paper_2303_04390_b200/csrc/schedule.cpp
