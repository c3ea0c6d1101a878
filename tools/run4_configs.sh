R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
$R --master-port 29521 bench.py --gpus 4 --qubits 32 --steps 1 --warmup 1 > gpurun_out/b32_gf_flat_n4.json 2> gpurun_out/b32_gf_flat_n4.err
$R --master-port 29522 bench.py --gpus 4 --qubits 32 --schedule adhoc --steps 1 --warmup 1 > gpurun_out/b32_gf_adhoc_n4.json 2> gpurun_out/b32_gf_adhoc_n4.err
$R --master-port 29523 bench.py --gpus 4 --qubits 34 --circuit hea --steps 1 --warmup 1 > gpurun_out/b34_hea_n4.json 2> gpurun_out/b34_hea_n4.err
$R --master-port 29524 bench.py --gpus 4 --qubits 30 --circuit hea --hamiltonian uniform --terms 1000 --steps 1 --warmup 1 > gpurun_out/b30_uni_n4.json 2> gpurun_out/b30_uni_n4.err
