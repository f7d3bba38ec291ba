# ring depth vs per-step latency of the small-S traversal (dengue tree)
for f in "" paper_2303_04390_b200/lib/libphylograd_vD2.so paper_2303_04390_b200/lib/libphylograd_vD8.so paper_2303_04390_b200/lib/libphylograd_vD16.so; do
  echo "== ${f:-default D=4}"
  if [ -n "$f" ]; then export PHYLOGRAD_LIB=$PWD/$f; else unset PHYLOGRAD_LIB; fi
  timeout 300 python scripts/scan_patterns.py 148 1184 4736 10000 2>&1 | tail -4
done
