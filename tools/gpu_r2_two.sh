bash tools/gpu_r2_dropin_vgg.sh
bash tools/gpu_r2_profile.sh
cat gpurun_out/r2_prof_stage.csv gpurun_out/r2_prof_small.csv | cut -c1-400 | head -30
