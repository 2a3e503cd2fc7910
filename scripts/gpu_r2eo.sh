# Halo exchange: stream fork and fused receive ablations (processes, N=2), and their effect on the SpMV overlap
O=gpurun_out; mkdir -p $O
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --nproc-per-node 2"
p=29890
for v in default nofork nofuse nofork_nofuse; do
  env=""
  case $v in nofork) env="SFG_P2P_NO_FORK=1";; nofuse) env="SFG_P2P_NO_FUSED_UNPACK=1";; nofork_nofuse) env="SFG_P2P_NO_FORK=1 SFG_P2P_NO_FUSED_UNPACK=1";; esac
  p=$((p+1)); env $env timeout 300 $TR --master-port $p bench_configs.py --config 2 > $O/r2eo_halo_$v.log 2>&1
  p=$((p+1)); env $env timeout 300 $TR --master-port $p bench_configs.py --config 3 --spmv > $O/r2eo_spmv_$v.log 2>&1
  p=$((p+1)); env $env timeout 300 $TR --master-port $p bench_configs.py --config 2 --n2 2048 --steps 10 > $O/r2eo_halo2048_$v.log 2>&1
done
