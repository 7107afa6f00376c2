for tl in 256 512 768 1024 1536; do echo "stages=2 tile=$tl"; BF_TMA_STAGES=2 BF_TMA_TILE=$tl python tools/profile_step.py --config 3 --maxit 60 --warm 2 2>&1 | tail -1 | cut -c1-60; done
