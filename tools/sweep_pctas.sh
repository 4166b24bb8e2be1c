for c in 1 2 3 4 5; do echo "pctas=$c"; PTROM_FOM_PCTAS=$c python tools/fom_time_probe.py | tail -1; done
