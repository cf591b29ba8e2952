# the reference's acceptance runner: unmodified (CPU) and relinked against the drop-in
mkdir -p gpurun_out/acceptance
for b in acceptance_ref acceptance_gpu acceptance_gpu_full; do
  ./oracle/_ref/$b > gpurun_out/acceptance/$b.txt 2>&1; echo "$b exit=$? (failures)" >> gpurun_out/acceptance/$b.txt
done
