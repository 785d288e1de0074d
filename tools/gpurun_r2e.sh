python -c "
import ctypes as C, numpy as np, time
from paper_2605_02953_b200 import _lib
import torch; torch.cuda.init()
out=(C.c_uint8*256)(); n=C.c_int()
t=time.time(); _lib.call('tf_sm_die_map', 0, out, 256, C.byref(n)); dt=time.time()-t
a=np.frombuffer(out, np.uint8)[:n.value]; print('n_sms', n.value, 'die0', int((a==0).sum()), 'die1', int((a==1).sum()), 'probe s', round(dt,3)); print(a.tolist())
" > gpurun_out/r2e_diemap_lib.txt 2>&1
for m in 1 2; do
  TF_GEMM_DIE=$m timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_fullsize.py -q -x -k "not ipc" > gpurun_out/r2e_gemmtest_die$m.txt 2>&1; echo "rc=$?" >> gpurun_out/r2e_gemmtest_die$m.txt
done
bash tools/gemm_l2_probe.sh "TF_GEMM_DIE=0" "TF_GEMM_DIE=1" "TF_GEMM_DIE=2" "TF_GEMM_DIE=2 TF_GEMM_KSNAKE=1"
