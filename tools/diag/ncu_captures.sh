#!/bin/bash
# ncu --set full captures of single full-size kernel launches (one per
# config), exported to text on the box (reports are too large to bring back).
# usage: ncu_captures.sh [name:regex:config:what ...]
mkdir -p gpurun_out/ncu
N="ncu -f --set full --clock-control none --import-source on"
specs=("$@")
if [ ${#specs[@]} -eq 0 ]; then
  specs=(k3_c2:condense6_kernel:C2:none k3_c4:condense6_kernel:C4:none k3_c3:condense5_kernel:C3:none
         k6_c5:postprocess2_kernel:C5:post k4_c2:scatter_faces:C2:scatter k7_c4:convection_kernel:C4:conv
         k2_c2:quad_build:C2:none k5_c2:recover3:C2:none)
fi
for s in "${specs[@]}"; do
  IFS=: read name rx cfg what <<< "$s"
  $N -k regex:$rx -c 1 -o /tmp/$name python tools/diag/run_config.py $cfg $what > gpurun_out/ncu/$name.log 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/ncu/${name}_details.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_source.csv 2>&1
  gzip -c /tmp/${name}_source.csv > gpurun_out/ncu/${name}_source.csv.gz
  ncu -i /tmp/$name.ncu-rep --page raw --csv > /tmp/${name}_raw.csv 2>&1
  gzip -c /tmp/${name}_raw.csv > gpurun_out/ncu/${name}_raw.csv.gz
done
ls -la gpurun_out/ncu
