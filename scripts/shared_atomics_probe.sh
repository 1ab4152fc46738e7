# Which shared-memory atomics are native on sm_100a?  (Evidence for DESIGN.md §6:
# a V-side fp32 codeword histogram would need fp32 shared atomics.)
nvcc -gencode arch=compute_100a,code=sm_100a -cubin -o /tmp/shared_atomics_probe.cubin \
  "$(dirname "$0")/shared_atomics_probe.cu" && cuobjdump -sass /tmp/shared_atomics_probe.cubin | grep -E "ATOMS|RED"
