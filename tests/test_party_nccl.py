"""Party mode over NCCL: three ranks, one GPU per party, every
share and ledger checked against the oracle by tools/party_nccl.py --check.
Runs where >= 3 GPUs are visible (gpurun --gpus 4); skipped otherwise."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 3, reason="needs 3 GPUs")
@pytest.mark.parametrize("backend,variant", [("shamir", "mpc-lift"), ("replicated", "mpc-lift"),
                                             ("shamir", "plain-mask"), ("replicated", "no-lift")])
def test_party_mode_over_nccl(backend, variant):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="0,1,2")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "3",
           "--master-addr", "127.0.0.1", "--master-port", str(29541 + hash((backend, variant)) % 50),
           os.path.join(ROOT, "tools", "party_nccl.py"), "--check", "--backend", backend, "--variant", variant]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    assert line["check"] == {"person_match": True, "row_bits": True, "ledgers": True}
    assert line["person_match"][0] == 1
