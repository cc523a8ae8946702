# A/B one experiment build (V=path to .so, TAG): core parity tests, determinism, 2 alternating bench passes
V=${V:-paper_2601_22275_b200/libvmb_x.so}; TAG=${TAG:-x}
VMB_LIB=$PWD/$V timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_precision.py tests/test_gpu_fuzz.py tests/test_gpu_known_answers.py -x -q --timeout 300 -m "gpu and not slow" > gpurun_out/${TAG}_bn128_pytest.log 2>&1; tail -2 gpurun_out/${TAG}_bn128_pytest.log
VMB_LIB=$PWD/$V python scripts/diag_determinism.py 4 > gpurun_out/${TAG}_det.txt 2>&1; grep -c "bad/rows (0," gpurun_out/${TAG}_det.txt
bash scripts/abn.sh 2 paper_2601_22275_b200/libvmb.so $V
