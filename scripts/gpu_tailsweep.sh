for t in 3 4 5 6 8; do echo "TAIL_MAX=$t"; DM_TAIL_MAX=$t python scripts/prof_step.py c5 3 2>&1 | grep -E "config5|count  *[0-9.]*ms write   0.000" | cut -c1-200; done
