# retune after the round-2 changes: service threshold and CTA cache slots (time_enum: S28 full, S32 2^24 block)
for th in 10 12 14 16 18 20 22; do
  echo "thresh $th" >> gpurun_out/r2s83.log
  TV_SERVICE_THRESH=$th python tools/time_enum.py >> gpurun_out/r2s83.log 2>&1
done
for cs in 128 512; do
  echo "cta_slots $cs" >> gpurun_out/r2s83.log
  TV_CTA_SLOTS=$cs python tools/time_enum.py >> gpurun_out/r2s83.log 2>&1
done
echo "default" >> gpurun_out/r2s83.log
python tools/time_enum.py >> gpurun_out/r2s83.log 2>&1
