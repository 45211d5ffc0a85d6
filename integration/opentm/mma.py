"""The reference's MMA optimizer (mma.py, minimum-volume model) is outside the B200
hot path (not in north_star; the reference itself caps it at
64^3).  The names exist so ``from opentm.mma import ...`` resolves; using them
raises."""


class MMAState:
    def __init__(self, *args, **kwargs):
        raise NotImplementedError("the MMA optimizer is not part of the B200 build (model 'oc' only)")


def mma_update(*args, **kwargs):
    raise NotImplementedError("the MMA optimizer is not part of the B200 build (model 'oc' only)")
