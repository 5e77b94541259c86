python scripts/probe_config4.py --scale 0.5 --steps 4 2>&1 | grep '"step": 3' | cut -c1-300
python scripts/round_phases.py --config 4 --scale 0.25 2>&1 | tail -11
