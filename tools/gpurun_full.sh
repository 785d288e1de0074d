timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/full_test.txt 2>&1
echo "rc=$?" >> gpurun_out/full_test.txt
