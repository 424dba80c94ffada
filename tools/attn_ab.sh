mkdir -p gpurun_out/at2
for v in s3 s4 def; do
  if [ $v = def ]; then L=paper_2311_04934_b200/lib/libpcb200.so; else L=paper_2311_04934_b200/lib/libpcb200_$v.so; fi
  for rep in 1 2; do PCB_LIB_PATH=$L timeout 120 python tools/attn_probe.py >> gpurun_out/at2/$v.txt 2>&1; done
done
