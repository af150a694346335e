# ncu on the headline list and the two other configs; the reports are reduced
# to CSV summaries on the box (gpurun copies back <= 64 MiB).
bash tools/gpu_ncu_headline.sh > gpurun_out/ncu_run.log 2>&1
for r in llama8b resnet_sgd gpt2; do
  ncu -i gpurun_out/ncu_full_$r.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$r.csv 2>/dev/null
  ncu -i gpurun_out/ncu_full_$r.ncu-rep --page details --csv > gpurun_out/ncu_details_$r.csv 2>/dev/null
done
ncu -i gpurun_out/ncu_full_llama8b.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_sass_llama8b.csv 2>/dev/null
gzip -f gpurun_out/ncu_sass_llama8b.csv
rm -f gpurun_out/ncu_full_resnet_sgd.ncu-rep gpurun_out/ncu_full_gpt2.ncu-rep
gzip -f gpurun_out/ncu_full_llama8b.ncu-rep
ls -la gpurun_out/ | head -40
