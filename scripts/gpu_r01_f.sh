mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
for d in 2 3 4 5 6 7 8 9 10; do
  for k in 0 $((d-1)); do python -m paper_2501_03121_b200.cli tvc --dims paper:d$d --mode $k --iters 5 --peak 6372.5e9 2>&1 | tail -1; done
done > gpurun_out/cli_paper.csv; echo cli_rc=$?
python -m paper_2501_03121_b200.cli hopm --dims paper:d4 --split 3 --sweeps 2 --iters 2 --peak 6372.5e9 > gpurun_out/cli_hopm.csv 2>&1; echo hopm_rc=$?
python -m paper_2501_03121_b200.cli triad --dims 1073741824 --iters 10 --peak 6372.5e9 > gpurun_out/cli_triad.csv 2>&1; echo triad_rc=$?
