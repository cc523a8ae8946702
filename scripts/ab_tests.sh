# Core GPU tests on one library build (V) then an alternating bench A/B against B:
#   V=paper_2601_22275_b200/libvmb_x.so B=paper_2601_22275_b200/libvmb_base.so TAG=x bash scripts/ab_tests.sh
V=${V:-paper_2601_22275_b200/libvmb.so}; B=${B:-paper_2601_22275_b200/libvmb_base.so}; TAG=${TAG:-x}
VMB_LIB=$PWD/$V timeout -s KILL 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py \
  tests/test_gpu_precision.py tests/test_gpu_fuzz.py tests/test_gpu_known_answers.py tests/test_gpu_seq.py \
  tests/test_gpu_fp32_tc.py tests/test_gpu_multi.py -q --timeout 300 -x > gpurun_out/${TAG}_pytest.log 2>&1
tail -2 gpurun_out/${TAG}_pytest.log
VMB_LIB=$PWD/$V python scripts/diag_determinism.py 4 > gpurun_out/${TAG}_det.txt 2>&1; grep -c "bad/rows (0," gpurun_out/${TAG}_det.txt
bash scripts/abn.sh ${PASSES:-2} $B $V
