O=gpurun_out; mkdir -p $O
timeout 200 ./scripts/ll128_bench 10 > $O/r2r_ll128_trace.log 2>&1; echo "rc=$?" >> $O/r2r_ll128_trace.log
