#!/bin/bash
# Why does the driver's ncu launch census of smoke() fail on embed_kernel?
# Variants: as-is, eager module loading, PDL off, no green contexts, all off.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out/census
run() {
  name=$1; shift
  env "$@" timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv \
    --log-file gpurun_out/census/$name.csv python -c "import __graft_entry__ as g; g.smoke()" \
    > gpurun_out/census/$name.log 2>&1
  echo "$name rc=$? rb_launches=$(grep -c 'rb::\|_kernel' gpurun_out/census/$name.csv)"
}
run base
run eager CUDA_MODULE_LOADING=EAGER
run nopdl RB_PDL=0
run nogreen RB_SMOKE_SPLIT=none
run nogreen_nopdl RB_SMOKE_SPLIT=none RB_PDL=0
