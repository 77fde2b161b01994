mkdir -p gpurun_out; : > gpurun_out/ablate.log
for ab in 0 63 127 255 64 128 192; do
  LFMMI_ABLATE=$ab python scripts/prof_sections.py 2>&1 | grep -E "TOTAL|ablate=" >> gpurun_out/ablate.log
done
