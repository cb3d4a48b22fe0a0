set -x
python scripts/timeline.py 5
DDM_SERIAL=1 python scripts/timeline.py 5
python scripts/timeline.py 3
DDM_SERIAL=1 python scripts/timeline.py 3
DDM_PDL=0 python scripts/timeline.py 3
python scripts/timeline.py 4
DDM_SERIAL=1 python scripts/timeline.py 4
