"""Rank-group (one process per GPU) hot path vs the single-process run of
the same partitions: bitwise SpMV, PCG, assembly and simulation state.

On a 1-GPU box both ranks share cuda:0 (time-sliced contexts; the peer
windows are CUDA IPC mappings of the same device), which exercises the
same flag / peer-load protocol as an NVLink multi-GPU node."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from oracle_bindings import ORACLE

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn(world, parts, out_dir, timeout=600):
    port = free_port()
    procs = []
    for r in range(world):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE=str(world), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   WEFT_DEVICE="0", WEFT_PARTS=str(parts), LOCAL_RANK=str(r))
        procs.append(subprocess.Popen([sys.executable, os.path.join(HERE, "mp_rank.py"), str(out_dir)], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=timeout)[0])
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-4000:]
    return [dict(np.load(os.path.join(out_dir, f"rank{r}.npz"))) for r in range(world)]


@pytest.fixture(scope="module")
def weft():
    from paper_2008_00409_b200 import weft as w
    return w


@pytest.mark.parametrize("world,parts", [(2, 2), (2, 4), (4, 4)])
def test_rank_group_matches_single_process(weft, tmp_path, world, parts):
    import mp_rank

    ranks = spawn(world, parts, tmp_path)
    single, engines = mp_rank.run(lambda: weft.Engine(parts), 1, 0, lambda e: None)
    for e in engines:
        e.close()
    pr = mp_rank.problems()
    s = pr["spmv"]
    bounds = weft.make_partitions(s.rows, parts)
    span = parts // world
    y_or = ORACLE.spmv(s, pr["x"], parts)
    for r, res in enumerate(ranks):
        b, e = bounds[r * span][0], bounds[(r + 1) * span - 1][1]
        sl = slice(3 * b, 3 * e)
        assert np.array_equal(res["spmv_y"][sl], y_or[sl])
        assert np.array_equal(res["spmv_y2"][sl], single["spmv_y2"][sl])
    # PCG: identical scalars on every rank -> identical iterations/history
    pb = weft.make_partitions(pr["spd"].rows, parts)
    for r, res in enumerate(ranks):
        b, e = pb[r * span][0], pb[(r + 1) * span - 1][1]
        assert int(res["pcg_iterations"]) == int(single["pcg_iterations"])
        assert np.array_equal(res["pcg_hist"], single["pcg_hist"])
        assert np.array_equal(res["pcg_x"][3 * b:3 * e], single["pcg_x"][3 * b:3 * e])
    # assembly: each rank's rows are the single-process matrix's rows
    srp, scols, svals = single["asm_row_ptr"], single["asm_cols"], single["asm_vals"]
    for res in ranks:
        f = int(res["asm_first_row"])
        rp = res["asm_row_ptr"]
        nloc = len(rp) - 1
        k0, k1 = srp[f], srp[f + nloc]
        assert np.array_equal(rp, srp[f:f + nloc + 1] - k0)
        assert np.array_equal(res["asm_cols"], scols[k0:k1])
        assert np.array_equal(res["asm_vals"], svals[k0:k1])
        assert np.array_equal(res["asm_rhs"], single["asm_rhs"][3 * f:3 * (f + nloc)])
    for r, res in enumerate(ranks):
        f = int(res["asm_first_row"])
        nloc = len(res["asm_row_ptr"]) - 1
        assert int(res["asm_pcg_its"]) == int(single["asm_pcg_its"])
        assert np.array_equal(res["asm_pcg_x"][3 * f:3 * (f + nloc)], single["asm_pcg_x"][3 * f:3 * (f + nloc)])
    # device-resident steps: full replicated state bitwise, candidate shares
    for res in ranks:
        assert "sim_error" not in res, str(res["sim_error"])
    for res in ranks:
        assert np.array_equal(res["sim_x"], single["sim_x"])
        assert np.array_equal(res["sim_v"], single["sim_v"])
        assert np.array_equal(res["sim_its"], single["sim_its"])
    assert np.array_equal(sum(r["sim_dcd"] for r in ranks), single["sim_dcd"])
    assert np.array_equal(sum(r["sim_ccd"] for r in ranks), single["sim_ccd"])
    # whole steps with contacts and impact zones: the merged collide gives
    # every rank the single-process proximities / impacts, and the contact
    # columns that cross the cut go through the PCG's peer-memory halo
    assert single["con_counts"].shape[0] >= 2 and single["con_counts"][:, 1].min() > 50, \
        (single["con_counts"], str(single.get("con_error")))
    for res in ranks:
        if "con_error" in single:
            assert str(res.get("con_error")) == str(single["con_error"])
        else:
            assert "con_error" not in res, str(res["con_error"])
        assert np.array_equal(res["con_counts"], single["con_counts"])
        assert np.array_equal(res["con_x"], single["con_x"])
        assert np.array_equal(res["con_v"], single["con_v"])
