# every --workload sweep line of bench.py at N = 1/2/4 (builder evidence for BASELINE configs[1..3])
O=gpurun_out/cli; mkdir -p $O
run() { n=$1; shift; timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2967$n bench.py --gpus $n "$@"; }
run 2 --workload p2p --steps 20 > $O/p2p_n2.jsonl 2> $O/p2p_n2.err
for n in 2 4; do for w in allreduce bcast; do run $n --workload $w --steps 20 > $O/${w}_n$n.jsonl 2> $O/${w}_n$n.err; done; done
timeout 900 python bench.py --workload dgemm --steps 3 > $O/dgemm_n1.jsonl 2> $O/dgemm_n1.err
for n in 2 4; do run $n --workload dgemm --steps 3 > $O/dgemm_n$n.jsonl 2> $O/dgemm_n$n.err; done
