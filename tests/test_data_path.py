"""Device-side data path: band masks / pixel lists built on the
device (dilation_band + generate_rays' pixel lists, render.cpp:17-45, 57-66) and
the device box-union RGB-D renderer (twin of scenes.box_union_scene)."""
import numpy as np
import pytest

from paper_2503_01582_b200 import FieldArch, ObjectTrainer, TrainConfig, scenes

pytestmark = pytest.mark.gpu

ARCH = FieldArch(hash_levels=4, features_per_level=2, log2_table_size=10, base_resolution=4, per_level_scale=1.5,
                 hidden_width=16, hidden_layers=1)


def _masks(rng):
    H, W = 37, 53
    out = []
    m = np.zeros((H, W), np.uint8)
    m[10:20, 15:30] = 3
    out.append((m, 3, 8))
    out.append(((rng.random((H, W)) < 0.05).astype(np.uint8) * 2, 2, 3))  # speckle, instance 2
    m = np.zeros((H, W), np.uint8)
    m[0:5, W - 6:W] = 1  # touches the border
    m[H - 1, 0] = 1
    out.append((m, 1, 8))
    out.append((m, 1, 0))  # band_px 0 -> empty band
    out.append((m, 1, 1))
    out.append((np.ones((H, W), np.uint8), 1, 8))  # full: empty band
    return out


def test_device_pixel_lists_match_dilation_band(ctx, oracle):
    from paper_2503_01582_b200.trainer import Camera

    rng = np.random.default_rng(4)
    for mask, inst, band in _masks(rng):
        H, W = mask.shape
        cam = Camera(fx=40.0, fy=40.0, cx=W / 2, cy=H / 2, width=W, height=H)
        obj = ObjectTrainer.create(ctx, ARCH, grid_res=8, cfg=TrainConfig(band_px=band))
        obj.set_frames([cam], np.zeros((1, H, W, 3), np.float32), np.zeros((1, H, W), np.float32), mask[None],
                       instance_value=inst)
        _, _, op, bp = obj.get_frame(0)
        want_band = oracle.dilation_band(mask, inst, band)
        assert np.array_equal(op, np.flatnonzero(mask.reshape(-1) == inst))
        assert np.array_equal(bp, np.flatnonzero(want_band.reshape(-1)))
        obj.close()


def test_device_pixel_lists_match_reference(ctx, ref):
    from paper_2503_01582_b200.trainer import Camera

    rng = np.random.default_rng(5)
    for mask, inst, band in _masks(rng):
        H, W = mask.shape
        cam = Camera(fx=40.0, fy=40.0, cx=W / 2, cy=H / 2, width=W, height=H)
        obj = ObjectTrainer.create(ctx, ARCH, grid_res=8, cfg=TrainConfig(band_px=band))
        obj.set_frames([cam], np.zeros((1, H, W, 3), np.float32), np.zeros((1, H, W), np.float32), mask[None],
                       instance_value=inst)
        _, _, _, bp = obj.get_frame(0)
        assert np.array_equal(bp, np.flatnonzero(ref.dilation_band(mask, inst, band).reshape(-1)))
        obj.close()


def _scene(res=96, n=6, seed=3):
    rng = np.random.default_rng(seed)
    boxes = scenes.random_boxes(rng)
    cams = scenes.fibonacci_cameras(n, 1.5, res, res, float(res))
    return boxes, cams


def test_synth_frames_match_host_renderer(ctx):
    boxes, cams = _scene()
    host = scenes.box_union_scene(n_views=len(cams), res=cams[0].width, boxes=boxes)
    obj = ObjectTrainer.create(ctx, ARCH, grid_res=8, cfg=TrainConfig())
    obj.synth_frames(cams, boxes)
    for i in range(len(cams)):
        rgb, dep, op, bp = obj.get_frame(i)
        m_dev = np.zeros(dep.size, bool)
        m_dev[op] = True
        m_host = host.mask[i].reshape(-1) == 1
        agree = m_dev == m_host
        assert agree.mean() > 0.999, agree.mean()  # grazing pixels may differ by one rounding
        both = (m_dev & m_host).reshape(dep.shape)
        np.testing.assert_allclose(dep[both], host.depth[i][both], rtol=2e-5, atol=1e-6)
        same_box = np.all(rgb == host.rgb[i], axis=-1)
        assert same_box[both].mean() > 0.999  # the nearest box agrees except at box seams
        assert not dep[~m_dev.reshape(dep.shape)].any() and not rgb[~m_dev.reshape(dep.shape)].any()
        band = np.zeros(dep.size, bool)
        band[bp] = True
        assert not (band & m_dev).any() and band.any()
    obj.close()


def test_synth_noise_and_missing_statistics(ctx):
    boxes, cams = _scene(res=256, n=2)
    clean = ObjectTrainer.create(ctx, ARCH, grid_res=8)
    noisy = ObjectTrainer.create(ctx, ARCH, grid_res=8)
    clean.synth_frames(cams, boxes)
    noisy.synth_frames(cams, boxes, depth_noise=0.01, missing_frac=0.05, seed=9)
    for i in range(2):
        _, d0, op0, _ = clean.get_frame(i)
        _, d1, op1, _ = noisy.get_frame(i)
        assert np.array_equal(op0, op1)  # mask = hit, noise does not move it
        hit = d0.reshape(-1)[op0]
        got = d1.reshape(-1)[op0]
        miss = got == 0
        assert abs(miss.mean() - 0.05) < 0.01, miss.mean()
        err = (got - hit)[~miss]
        assert abs(err.mean()) < 1e-3 and abs(err.std() - 0.01) < 1e-3, (err.mean(), err.std())
    # deterministic per seed
    again = ObjectTrainer.create(ctx, ARCH, grid_res=8)
    again.synth_frames(cams, boxes, depth_noise=0.01, missing_frac=0.05, seed=9)
    assert np.array_equal(again.get_frame(1)[1], noisy.get_frame(1)[1])
    for o in (clean, noisy, again):
        o.close()


def test_training_on_device_frames_equals_host_upload(ctx):
    """Frames rendered on the device train exactly like the same pixels uploaded from the host."""
    boxes, cams = _scene(res=64, n=4)
    cfg = TrainConfig(rays_per_iter=256, samples_per_ray=16, prior_sampling=0, grid_refresh_every=0)
    a = ObjectTrainer.create(ctx, ARCH, grid_res=8, seed=5, cfg=cfg)
    a.synth_frames(cams, boxes, depth_noise=0.01, missing_frac=0.05, seed=2)
    rgb, dep, masks = [], [], []
    for i in range(len(cams)):
        r, d, op, _ = a.get_frame(i)
        m = np.zeros(d.size, np.uint8)
        m[op] = 1
        rgb.append(r), dep.append(d), masks.append(m.reshape(d.shape))
    b = ObjectTrainer.create(ctx, ARCH, grid_res=8, seed=5, cfg=cfg)
    b.set_frames(cams, np.stack(rgb), np.stack(dep), np.stack(masks), 1)
    la, lb = a.train_step(5), b.train_step(5)
    for x, y in zip(la, lb):
        assert x["frame"] == y["frame"] and x["n_samples"] == y["n_samples"]
        assert abs(x["total"] - y["total"]) <= 1e-6 * abs(y["total"])
    a.close()
    b.close()
