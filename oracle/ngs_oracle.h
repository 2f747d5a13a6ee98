/* placeholder: the C restatement of the reference path is built in a later step */
