# ncu --set full of k_chunk (round 1) and k_sims (round 1) of a config-2 search, summarised
mkdir -p gpurun_out
for k in k_chunk k_sims; do
ncu --profile-from-start off --set full --import-source on --clock-control none \
  --kernel-name regex:"$k" --launch-skip 1 --launch-count 1 \
  -o gpurun_out/full_$k -f python tools/prof_search.py --engine 0 > gpurun_out/ncu_$k.log 2>&1
python tools/ncu_summary.py gpurun_out/full_$k.ncu-rep gpurun_out/full_$k.json > /dev/null 2>&1
cat gpurun_out/full_$k.json
ncu -i gpurun_out/full_$k.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/src_$k.csv 2>/dev/null
python tools/src_hot.py gpurun_out/src_$k.csv 2>&1 | head -60
done
rm -f gpurun_out/*.ncu-rep
