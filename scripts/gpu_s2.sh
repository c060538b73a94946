exec > gpurun_out/s2b.log 2>&1
python scripts/ovh_probe.py c2
python scripts/ovh_probe.py c4
