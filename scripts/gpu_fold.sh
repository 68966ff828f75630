mkdir -p gpurun_out/ncu_fold
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider -k "fold or ring or dtvc or reduce or mixed or hopm" > gpurun_out/pytest_fold.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/pytest_fold.log
python scripts/util_one.py > gpurun_out/ncu_fold/plain.log 2>&1 && \
ncu --set full --clock-control none -k regex:"k_fold" -s 2 -c 2 -o /tmp/p_fold python scripts/util_one.py > gpurun_out/ncu_fold/ncu.log 2>&1; echo ncu_rc=$?
ncu -i /tmp/p_fold.ncu-rep --page details --csv > gpurun_out/ncu_fold/details.csv 2>/dev/null
