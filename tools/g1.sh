timeout 1200 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
bash tools/profile_round.sh r01b 2>&1 | tail -15
