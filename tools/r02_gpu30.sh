# round-2 evidence refresh: launch list + --set full of the current kernels, then the per-kernel full captures
bash tools/make_profiles.sh r02
bash tools/r02_prof1.sh
