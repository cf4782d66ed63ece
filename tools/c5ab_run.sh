# A/B of the C5 path over the libraries named on the command line
# (default = the in-tree libfrr.so, else tools/variants/libfrr_<name>.so)
mkdir -p gpurun_out
for v in "$@"; do
  if [ $v = default ]; then L=paper_2501_07642_b200/libfrr.so; else L=tools/variants/libfrr_$v.so; fi
  FRR_LIBRARY=$L timeout 120 python tools/c5_ab.py $v >> gpurun_out/c5ab.jsonl 2>>gpurun_out/c5ab.err
done
