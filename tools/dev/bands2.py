"""Config-2 page: device time per call against the forced band count (dev)."""
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
import paper_1905_13038_b200 as ab  # noqa: E402

H, W = 3300, 2550
xs = torch.zeros((8, H, 2560), dtype=torch.uint8, device="cuda")
xs[:, :, :W] = torch.from_numpy(synth.page(H, W, synth.config_seed(2, 0))).cuda()
outs = torch.empty((8, H, W), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
for hw in (15, 31, 63, 127, 255):
    row = {"hw": hw}
    for nb in ("", "25", "50", "100", "200", "400", "800"):
        if nb:
            os.environ["ABIN_V4_BANDS"] = nb
        else:
            os.environ.pop("ABIN_V4_BANDS", None)
        for i in range(3):
            ab.sauvola(xs[i, :, :W], hw, hw, out=outs[i])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(2e8))
        a.record(st)
        for i in range(40):
            ab.sauvola(xs[i % 8, :, :W], hw, hw, out=outs[i % 8])
        b.record(st)
        torch.cuda.synchronize()
        row[nb or "model"] = round(a.elapsed_time(b) / 40 * 1e3, 1)
    print(json.dumps(row))
