# time each experimental variant on the dengue traversal
for f in paper_2303_04390_b200/lib/libphylograd_v*.so; do
  echo "== $f"; PHYLOGRAD_LIB=$PWD/$f timeout 300 python scripts/scan_patterns.py ${SCAN_C:-10000} 2>&1 | tail -3
done
