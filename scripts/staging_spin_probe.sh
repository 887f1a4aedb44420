for sp in 0 20000; do PI0B_STAGING_SPIN_US=$sp timeout 300 python scripts/staging_probe.py 3 7 | sed "s/^/spin $sp: /"; done
