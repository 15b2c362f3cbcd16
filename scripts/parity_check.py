"""Parity diagnostics: GPU library vs the C oracle on a workload (prints stats).

python scripts/parity_check.py [workload] [frames] [mode]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_00291_b200 as svx  # noqa: E402
from paper_2412_00291_b200 import workload as W  # noqa: E402
from oracle.bindings import OracleMap, parse_svox1  # noqa: E402


def compare_maps(gb, ob, tag):
    hg, kg, tg, sg = parse_svox1(gb)
    ho, ko, to, so = parse_svox1(ob)
    print(f"[{tag}] blocks gpu={len(kg)} oracle={len(ko)} keys_equal={np.array_equal(kg, ko)}")
    if not np.array_equal(kg, ko):
        return False
    w_eq = np.array_equal(tg["weight"], to["weight"])
    obs_g, obs_o = tg["weight"] > 0, to["weight"] > 0
    dd = np.abs(tg["distance"] - to["distance"])
    dg = np.abs(tg["gradient"] - to["gradient"]).max(axis=-1)
    print(f"[{tag}] observed gpu={obs_g.sum()} oracle={obs_o.sum()} same_set={np.array_equal(obs_g, obs_o)} "
          f"W_exact={w_eq} (mismatch {(tg['weight'] != to['weight']).sum()})")
    print(f"[{tag}] D max|diff|={dd.max():.3g} bit-exact frac={(tg['distance'] == to['distance']).mean():.6f} "
          f"G max|diff|={dg.max():.3g} bytes_equal={gb == ob}")
    sem_eq = sorted(sg) == sorted(so) and all(np.array_equal(sg[k], so[k]) for k in sg)
    if sg or so:
        mx = max((np.abs(sg[k] - so[k]).max() for k in sg if k in so), default=0.0)
        print(f"[{tag}] sem layers gpu={len(sg)} oracle={len(so)} bit-exact={sem_eq} max|diff|={mx:.3g}")
    return w_eq and dd.max() <= 1e-5 and dg.max() <= 1e-5


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    frames = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    modes = [int(sys.argv[3])] if len(sys.argv) > 3 else [1, 0]
    wl = W.make(name, frames)
    cfg = svx.MapConfig(wl.voxel_size, wl.truncation, wl.num_labels, 1 << 20)
    scans = [(p.numpy(), i) for p, i in wl.scans()]
    ok = True
    for mode in modes:
        icfg = svx.IntegratorConfig(mode=mode)
        g = svx.VoxelStore(cfg, 0)
        o = OracleMap(cfg)
        ti = svx.TsdfIntegrator(g, icfg)
        si = svx.SemanticIntegrator(g)
        for p, i in scans:
            pose = wl.pose(i)
            img = svx.project_cloud(p, pose, wl.model, g)
            d, h, n, v, dr = OracleMap.project(wl.model, p, pose)
            pe = (np.array_equal(img.depth, d), np.array_equal(img.height, h),
                  np.array_equal(img.normals, n), np.array_equal(img.normal_valid, v), img.dropped == dr)
            t0 = time.time()
            rg = ti.integrate_cloud(p, pose, wl.model)
            t1 = time.time()
            ro = o.integrate(wl.model, d, n, v, pose, icfg)
            t2 = time.time()
            print(f"mode={mode} frame={i} pts={len(p)} proj_exact={pe} gpu(upd={rg.updated_voxels}, new={rg.new_blocks}, "
                  f"{(t1-t0)*1e3:.1f} ms) oracle(upd={ro.updated_voxels}, new={ro.new_blocks}, {(t2-t1)*1e3:.0f} ms)")
            ok &= all(pe) and (rg.updated_voxels, rg.new_blocks) == (ro.updated_voxels, ro.new_blocks)
            for li in wl.label_images(i):
                a = si.integrate_labels(li)
                b = o.integrate_labels(li, svx.SemanticConfig())
                print(f"   labels upd gpu={a.updated_voxels} oracle={b.updated_voxels} ({a.elapsed_ms:.2f} ms)")
                ok &= a.updated_voxels == b.updated_voxels
        ok &= compare_maps(g.save_bytes(), o.save_bytes(), f"mode{mode}")
        dg = g.take_dirty_blocks(0)
        do = o.take_dirty(0)
        print(f"dirty tsdf equal: {np.array_equal(dg, do)} ({len(dg)})")
        g.close()
    print("PARITY", "OK" if ok else "FAIL", "launches", svx.kernel_launches())


if __name__ == "__main__":
    main()
