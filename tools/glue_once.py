"""One launch of each glued pass at the config-5 body shape (dev tool for ncu captures / C1D_PROFILE):
python tools/glue_once.py [fwd|fwd_skip|bwd|bwd_gadd]..."""
import os
import sys

which = sys.argv[1:] or ["fwd"]
sys.argv = [sys.argv[0], "64", "60000"]
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "time_glue.py")).read().split("def timeit")[0]
exec(src)
torch.cuda.synchronize()  # noqa: F821
calls = {
    "fwd": lambda: conv_forward_glued(x, w, p, bias=b, act_bf16=act_b, act_pad=pad, mask=mask),  # noqa: F821
    "fwd_skip": lambda: conv_forward_glued(x, w, p, bias=b, skip=skip, act=act, act_bf16=act_b, act_pad=pad,  # noqa
                                           mask=mask),  # noqa: F821
    "bwd": lambda: conv_backward_data_glued(dy, w, p, pad, q, mask=mask, grad_pre_bf16=gp, bias_grad=db),  # noqa
    "bwd_gadd": lambda: conv_backward_data_glued(dy, w, p, pad, q, gadd=gadd, mask=mask, gsum=gsum,  # noqa: F821
                                                 grad_pre_bf16=gp, bias_grad=db),  # noqa: F821
    "plain": lambda: cv.conv1d_forward(x, w, p, out=y),  # noqa: F821
}
for name in which:
    print(name, flush=True)
    calls[name]()
    torch.cuda.synchronize()  # noqa: F821
