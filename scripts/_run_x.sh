timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
bash scripts/ab.sh libub_base.so libub.so
P=0.1 bash scripts/ab.sh libub_base.so libub.so 2>&1 | head -4
DIST=bimodal bash scripts/ab.sh libub_base.so libub.so 2>&1 | head -4
