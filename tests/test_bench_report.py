"""The GPU rows of the reference's bench report (paper_1707_05062_b200/
bench_report.py): CSV layout and precision exactly as
proj/tests/test_bench.cpp:91-124 pins them, correctness-before-timing with an
injected corrupted implementation (:75-89), and the GPU harness itself."""
import numpy as np
import pytest

from paper_1707_05062_b200 import bench_report as br


def split_lines(csv):
    lines = csv.split("\n")
    assert lines[-1] == ""
    return lines[:-1]


def test_csv_layout_and_published_gain_example():
    rep = br.BenchReport("lenna", 512, 512, 1, 0, 8)
    rep.results.append(br.ImplTiming(br.DIRECT, [0.69], 0.69))
    rep.results.append(br.ImplTiming("gpu", [0.00546], 0.00546))
    lines = split_lines(br.write_report_csv(rep))
    assert lines == ["name,width,height,runs,median_s,run1_s,gain_vs_direct",
                     "gpu_direct,512,512,1,0.690000,0.690000,1.00",
                     "gpu,512,512,1,0.005460,0.005460,126.37"]


def test_csv_gain_empty_without_direct():
    rep = br.BenchReport("x", 8, 8, 2)
    rep.results.append(br.ImplTiming("gpu", [0.25, 0.5], 0.375))
    assert split_lines(br.write_report_csv(rep))[1] == "gpu,8,8,2,0.375000,0.250000,0.500000,"


def test_median_of_matches_reference():
    assert br.median_of([3.0, 1.0, 2.0]) == 2.0
    assert br.median_of([4.0, 1.0, 2.0, 3.0]) == 2.5


def test_refuses_to_time_a_corrupted_implementation(orc):
    rng = np.random.default_rng(12)
    img = rng.integers(0, 256, (16, 16), dtype=np.uint8)

    def good(a):
        from paper_1707_05062_b200 import ContrastCurve
        c = ContrastCurve()
        c.contrast_sum[:], c.cardinality[:] = orc.direct_curve(a)
        return c

    def bad(a):
        c = good(a)
        c.contrast_sum[10] += 1
        return c
    with pytest.raises(br.CurveMismatchError, match="t=10"):
        br.bench_image(img, [("direct", good), ("fast", bad)], runs=2, warmup=0)
    with pytest.raises(ValueError):
        br.bench_image(img, [("direct", good)], runs=0)
    with pytest.raises(ValueError):
        br.bench_image(img, ["gpu", "cpu"])  # unknown name


@pytest.mark.gpu
def test_gpu_rows(ctx):
    from paper_1707_05062_b200 import synth
    img = synth.generate("C1", device="cpu")[0].numpy()
    rep = br.bench_image(img, runs=3, warmup=1, image_id="C1")
    assert [t.name for t in rep.results] == [br.DIRECT, "gpu"]
    for t in rep.results:
        assert len(t.runs_s) == 3 and all(s > 0 for s in t.runs_s) and t.median_s > 0
    assert rep.gain_vs_direct(br.DIRECT) == pytest.approx(1.0)
    lines = split_lines(br.write_report_csv(rep))
    assert len(lines) == 3 and all(len(x.split(",")) == 5 + 3 + 1 for x in lines)


@pytest.mark.gpu
def test_gpu_video_rows(ctx, ref):
    import oracle
    from paper_1707_05062_b200 import synth
    frames = [f.numpy() for f in synth.generate("C3", device="cpu", n=3)]
    frames.insert(1, np.full_like(frames[0], 77))  # a constant frame passes through
    segs = []
    rep = br.bench_video(frames, ["gpu"], segmented_out=segs)
    assert rep.frame_count == 4 and rep.constant_frames == 1 and rep.results[0].fps > 0
    for f, s in zip(frames, segs):
        want, _, _ = oracle.ref_segment(ref, f, k=0)
        assert np.array_equal(s.pixels(), want)
