CFG=C4 TAG=c4 FR=20000 bash tools/gpu_prof_cfg.sh
CFG=C5 TAG=c5 FR=5000 bash tools/gpu_prof_cfg.sh
CFG=P TAG=p FR=5000 bash tools/gpu_prof_cfg.sh
CFG=C5 TAG=c5list FR=2000 KRE=fsscl EXTRA=--list bash tools/gpu_prof_cfg.sh
