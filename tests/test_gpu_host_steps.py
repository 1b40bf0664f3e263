"""GPU: Solver.host_steps (the host-resident trajectory the bench's e2e times) equals the
device-resident run bit for bit: the chunked, two-stream copies keep step i+1 reading
exactly step i's result (piece-wise event ordering), for RK4 and RK54, on the fused
tensor (c4) and simplex (c2) paths."""
import numpy as np
import pytest

from sdrt_inputs import CONFIGS, random_state

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,N", [("c4", (8, 4, 4)), ("c2", (6, 5))])
@pytest.mark.parametrize("chunks", [1, 3, 8])
@pytest.mark.parametrize("rk54", [False, True])
def test_host_steps_bitwise_device_run(name, N, chunks, rk54):
    from paper_2105_08632_b200.solver import Solver
    cfg = CONFIGS[name]
    S = Solver(cfg.etype, cfg.p, list(N), cfg.lo, cfg.hi, cfg.eq, device="cuda", **cfg.physics_kwargs())
    U0 = random_state(cfg, S.shape[0], S.K, seed=3, amp=0.2)
    steps = 5
    Ud = S.to_device(U0)
    (S.rk54_step if rk54 else S.rk_step)(Ud, cfg.dt, steps)
    ref = S.to_host(Ud)
    H = torch.empty(S.shape, dtype=torch.float64).pin_memory()
    H.copy_(S.to_device(U0).cpu())
    scratch = torch.empty(S.shape, dtype=torch.float64, device="cuda")
    S.host_steps(H, scratch, cfg.dt, steps, rk54=rk54, chunks=chunks)
    torch.cuda.synchronize()
    out = H[:, :, : S.K].numpy()
    S.close()
    assert np.array_equal(out, ref), np.abs(out - ref).max()
