timeout 2400 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
