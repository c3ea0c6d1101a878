#!/bin/bash
# Same-box A/B of a compile-time variant: the product libqrt.so vs LD_PRELOAD of
# paper_2410_04252_b200/libqrt_$VARIANT.so (built by build.build_variant), interleaved.
O=${OUT:-gpurun_out/r2var_${VARIANT}}; mkdir -p $O
V=$PWD/paper_2410_04252_b200/libqrt_${VARIANT}.so
for i in 1 2; do
  timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_base_$i.json 2>&1
  LD_PRELOAD=$V timeout 600 python bench.py --qubits 30 --no-cpu-baseline --steps 2 --warmup 3 > $O/gf30_var_$i.json 2>&1
  timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni_base_$i.json 2>&1
  LD_PRELOAD=$V timeout 600 python bench.py --qubits 30 --circuit hea --hamiltonian uniform --terms 4000 --no-cpu-baseline --steps 2 --warmup 3 > $O/uni_var_$i.json 2>&1
done
