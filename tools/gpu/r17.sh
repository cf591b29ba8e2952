# N > 1 code paths exercised on one GPU: torchrun world 1 with forced bands + forced all-reduce,
# the reference arm under torchrun, and the band path's launch accounting
set -u
python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 1 --steps 20 --warmup 5 --force-bands --force-reduce > gpurun_out/r17_bands.json 2> gpurun_out/r17_bands.err
echo "rc $?" >> gpurun_out/r17_bands.err
python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29612 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/r17_ref.json 2> gpurun_out/r17_ref.err
echo "rc $?" >> gpurun_out/r17_ref.err
tail -3 gpurun_out/r17_bands.err gpurun_out/r17_ref.err; cut -c1-600 gpurun_out/r17_bands.json; cut -c1-300 gpurun_out/r17_ref.json
