# end-of-round refresh on a 4-GPU box: full GPU suite, smoke, bench N=1/2/4 (+e2e),
# reference arm, launch list of the N=1 bench, ncu DRAM traffic of the N=1 stencil
mkdir -p gpurun_out
N=$(nvidia-smi -L | wc -l)
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/fin_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > gpurun_out/fin_bench_n1.log 2>&1; echo "bench n1 rc=$?"; tail -1 gpurun_out/fin_bench_n1.log | cut -c1-300
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference > gpurun_out/fin_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/fin_ref.log | cut -c1-200
for n in 2 4; do
  TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n"
  timeout 900 $TR bench.py --gpus $n > gpurun_out/fin_bench_n$n.log 2>&1; echo "bench n$n rc=$?"; tail -1 gpurun_out/fin_bench_n$n.log | cut -c1-300
done
B="python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu"
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/fin_launches.csv $B > gpurun_out/fin_ncu.log 2>&1; echo "ncu launches rc=$?"
CUDA_VISIBLE_DEVICES=0 timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:stencil_tma -s 3 -c 1 $B > gpurun_out/fin_ncu_traffic.txt 2>&1; echo "ncu traffic rc=$?"; grep -E "dram__|duration" gpurun_out/fin_ncu_traffic.txt
