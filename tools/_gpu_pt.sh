python -c "
import numpy as np; rng=np.random.default_rng(0); (rng.random((1024,1024,1024),dtype=np.float32)<0.02).astype(np.uint8).tofile('/tmp/b1024.raw')"
tools/pt_base /tmp/b1024.raw 1024 1024 1024 2>&1 | grep -E "kernel|pass"
