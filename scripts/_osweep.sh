for n in "1,1,1,1,1,1,1" "45,45,45,45,45,45,45" "16,16" "1,1" "45" "64,64,64,64,64,64,64,64"; do
  python scripts/gemm_sweep.py --knobs 8:200:0 --n $n 2>&1 | grep -E " o  .*members=[0-9]+ n=\[" | head -1
  python scripts/gemm_sweep.py --knobs 8:200:2 --n $n 2>&1 | grep -E " o  .*members=[0-9]+ n=\[" | head -1
done
