# single-GPU validation + refresh of every bench line (round-end style)
mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/fin/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -1 gpurun_out/fin/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.log 2>&1; echo smoke_rc=$?; tail -1 gpurun_out/fin/smoke.log
timeout 600 python scripts/tvc_modes_bench.py --set all > gpurun_out/fin/modes.jsonl 2>&1; echo modes_rc=$?
timeout 900 python bench.py > gpurun_out/fin/c2.json 2> gpurun_out/fin/c2.err; echo c2_rc=$?
for w in c1 c3 c4 c5; do
  timeout 900 python bench.py --workload $w --steps 10 --warmup 3 > gpurun_out/fin/$w.json 2> gpurun_out/fin/$w.err; echo ${w}_rc=$?
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin/ref.json 2> gpurun_out/fin/ref.err; echo ref_rc=$?
