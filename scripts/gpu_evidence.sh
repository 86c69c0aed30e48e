# the round's full evidence pass on one B200 (run under gpurun)
bash scripts/gpu_check.sh
bash scripts/gpu_configs.sh
bash scripts/gpu_profile.sh
