mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:codon_pmat -s 3 -c 1 -o gpurun_out/prof_pmat -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-flush --config 3 > gpurun_out/ncu_pmat.log 2>&1; tail -1 gpurun_out/ncu_pmat.log
python scripts/ncu_summary.py gpurun_out/prof_pmat.ncu-rep > gpurun_out/prof_pmat.txt; cat gpurun_out/prof_pmat.txt
python scripts/ncu_lines.py gpurun_out/prof_pmat.ncu-rep codon_pmat 25 > gpurun_out/prof_pmat_lines.txt 2>&1; head -25 gpurun_out/prof_pmat_lines.txt
rm -f gpurun_out/prof_pmat.ncu-rep
