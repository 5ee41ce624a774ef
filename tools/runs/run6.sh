python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02_gputests_6.log 2>&1; echo tests_rc=$?
tail -5 gpurun_out/r02_gputests_6.log
bash tools/runs/spmv_sweep.sh
