"""The C++ side of the drop-in boundary:
include/znn_gpu_engine.hpp compiled against the reference's own headers
(net_graph, engine<float>::sample_source, oracles.hpp) by tests/cpp/build.sh
and linked with libznn_cuda.so. One c1 round through znn::gpu_engine matches
the reference's double oracle round (tests/oracles.hpp:155-252) with the
updated parameters scattered back into net_graph<float>, and three further
rounds match the reference engine<float> (engine.hpp:65-254) loss by loss."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "gpu_engine_round")


@pytest.mark.parametrize("seed", [1, 7])
def test_gpu_engine_round_matches_reference(tmp_path, seed):
    from paper_1510_06706_b200 import configs
    assert os.path.exists(BIN), "oracle/_ref/gpu_engine_round is built by __graft_entry__.build()"
    cfg = configs.CONFIGS["c1"]
    spec = tmp_path / "c1.spec"
    spec.write_text(cfg.netspec())
    od = ",".join(map(str, cfg.out_dims))
    out = subprocess.run([BIN, str(spec), od, str(seed)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["ok"] and res["loss_err"] < 1e-4 and res["param_err"] < 1e-3, res
