set -x
for t in default 64,2,2 64,2,1 64,1,1; do
  if [ $t = default ]; then unset OC_CONV_TILE; else export OC_CONV_TILE=$t; fi
  timeout 300 python tools/conv_bench.py --shapes l1_3x3 --passes fprop,dgrad 2>&1 | sed "s/^/$t /"
done
unset OC_CONV_TILE
for cg in default 1 2; do
  if [ $cg = default ]; then unset OC_WGRAD_CG; else export OC_WGRAD_CG=$cg; fi
  timeout 300 python tools/conv_bench.py --shapes l1_3x3,r50_3x3_128 --passes wgrad 2>&1 | sed "s/^/wcg$cg /"
done
