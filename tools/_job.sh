O=gpurun_out
timeout 1500 python -m pytest tests/test_reference_driver_gpu.py tests/test_scale_gpu.py tests/test_krylov_gpu.py -m gpu -q -s --durations=15 > $O/newtests_r02.log 2>&1; echo "rc=$?" >> $O/newtests_r02.log
tail -40 $O/newtests_r02.log
