TF_GEMM_MC=1 timeout 600 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -x -q > gpurun_out/mc_test.txt 2>&1
echo "rc=$?" >> gpurun_out/mc_test.txt
bash tools/gemm_variants.sh "TF_GEMM_MC=0" "TF_GEMM_MC=1" "TF_GEMM_MC=1 TF_GEMM_KSNAKE=1"
