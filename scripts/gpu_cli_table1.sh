# the reference-style CSV (17 columns) for every mode of the paper's Table-1 tensors
mkdir -p gpurun_out
out=gpurun_out/cli_table1.csv
python -m paper_2501_03121_b200.cli tvc --dims paper:d2 --mode 0 --iters 5 --peak 6372.5e9 2>/dev/null | head -1 > $out
for d in 2 3 4 5 6 7 8 9 10; do
  for k in $(seq 0 $((d-1))); do
    python -m paper_2501_03121_b200.cli tvc --dims paper:d$d --mode $k --iters 5 --peak 6372.5e9 2>/dev/null | tail -1 >> $out
  done
done
echo rows=$(wc -l < $out)
python -m paper_2501_03121_b200.cli hopm --dims paper:d4 --split 3 --sweeps 2 --iters 2 --peak 6372.5e9 > gpurun_out/cli_hopm.csv 2>&1; echo hopm_rc=$?
python -m paper_2501_03121_b200.cli triad --dims 1073741824 --iters 10 --peak 6372.5e9 > gpurun_out/cli_triad.csv 2>&1; echo triad_rc=$?
