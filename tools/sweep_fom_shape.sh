# config-1 trajectory time over the persistent FOM kernel's CTA shape
# (threads per CTA x CTAs per SM x targets per thread); the PTROM_FOM_PROFILE
# line gives the phases.
for t in 128 256 512; do for c in 1 2 4; do for k in 2 4; do
  if [ $((t*c)) -le 1024 ]; then
    echo "tpb=$t pctas=$c tpt=$k"
    PTROM_FOM_TPB=$t PTROM_FOM_PCTAS=$c PTROM_FOM_TPT=$k python tools/fom_time_probe.py 2>&1 | tail -1
    PTROM_FOM_PROFILE=1 PTROM_FOM_TPB=$t PTROM_FOM_PCTAS=$c PTROM_FOM_TPT=$k python tools/fom_time_probe.py 2>&1 | grep fom_persistent | tail -1
  fi
done; done; done
