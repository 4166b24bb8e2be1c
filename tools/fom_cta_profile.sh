# per-CTA view of the persistent FOM's velocity phase (PTROM_FOM_PROFILE) over CTA shapes:
# "threads-per-CTA CTAs-per-SM targets-per-thread"
for cfg in "256 1 2" "256 2 2" "128 2 2" "128 4 2" "512 1 2" "128 3 2"; do set -- $cfg
  echo "tpb=$1 pctas=$2 tpt=$3"
  PTROM_FOM_TPB=$1 PTROM_FOM_PCTAS=$2 PTROM_FOM_TPT=$3 python tools/fom_time_probe.py 2>&1 | tail -1
  PTROM_FOM_PROFILE=1 PTROM_FOM_TPB=$1 PTROM_FOM_PCTAS=$2 PTROM_FOM_TPT=$3 python tools/fom_time_probe.py 2>&1 | grep -A1 fom_persistent | tail -2
done
