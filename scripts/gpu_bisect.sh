O=gpurun_out; mkdir -p $O; : > $O/bisect2.log
for i in 1 2 3; do
  echo "== device csr run $i" >> $O/bisect2.log
  timeout -s KILL 300 python -m pytest tests/test_gpu_multi.py -x -q >> $O/bisect2.log 2>&1; echo "rc $?" >> $O/bisect2.log
  echo "== host csr run $i" >> $O/bisect2.log
  SFG_HOST_CSR=1 timeout -s KILL 300 python -m pytest tests/test_gpu_multi.py -x -q >> $O/bisect2.log 2>&1; echo "rc $?" >> $O/bisect2.log
done
